"""Oracle: configuration space -- load, activity, validity, compact valid index (CVI).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions followed (readings in DESIGN.md §3):
  * features f_0..f_{d-1} in declaration order, finite ordered domains, default in domain
    (S:29-30 FeatureSpec);  activation predicate = conjunction of atomic comparisons over
    EARLIER features; a comparison involving an inactive feature is false
    (SURVEY ledger #8, "inactive exactly when its activation predicate is false").
  * raw index = mixed radix over digits, first-declared feature most significant
    ("deterministic order").
  * G1 canonical: an inactive feature carries its default digit ("default ... used when
    the feature is inactive"; SURVEY ledger #8).
  * G2/G3: the structural constraints of the preset (Table 1 gates P:507/P:510; S:109
    world-size rule; divisibility rules of Appendix B).
  * CVI position p = the p-th raw index, ascending, satisfying G1 and every non-resource
    constraint (reading R4).  The resource check (G4) is applied per candidate
    and lives in oracle/sim.py.

The CVI is computed here by a memoised dynamic program over features in declaration order
(count of valid completions of a prefix), NOT by the library's per-structure component
tables.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from functools import lru_cache

OPS = (">", ">=", "==", "!=", "<", "<=")


class SpaceError(ValueError):
    """Raised for invalid space documents (S:58 errors: schema, cycle, empty domain, unknown ref)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


@dataclass
class Atom:
    ref: int          # index of the referenced (earlier) feature
    op: str
    value: object     # python value compared against the referenced feature's value


@dataclass
class Feature:
    name: str
    kind: str
    values: list
    default_digit: int
    requires: list = field(default_factory=list)   # list[Atom]

    @property
    def n(self) -> int:
        return len(self.values)

    def numeric(self, digit):
        """Numeric encoding of a digit's value for the regression simulators (NEXT-1, reading
        R20): numbers as themselves, booleans 0/1, strings by their domain index."""
        v = self.values[digit]
        if isinstance(v, bool):
            return 1.0 if v else 0.0
        if isinstance(v, str):
            return float(digit)
        return float(v)


def _num(v):
    """Numeric view of a domain value: bools as 0/1 (S:452 'booleans as 0/1')."""
    if isinstance(v, bool):
        return 1 if v else 0
    return v


def compare(a, op, b) -> bool:
    """Atomic comparison value(ref) <op> value (S:29 'atomic comparisons, e.g. tp > 1')."""
    if isinstance(a, str) or isinstance(b, str):
        if op == "==":
            return a == b
        if op == "!=":
            return a != b
        raise SpaceError("schema", f"ordering comparison {op} on a categorical value")
    a, b = _num(a), _num(b)
    return {">": a > b, ">=": a >= b, "==": a == b, "!=": a != b, "<": a < b, "<=": a <= b}[op]


class Space:
    def __init__(self, doc: dict):
        self.doc = doc
        self.name = doc.get("name", "")
        self.sim_mode = doc.get("sim_mode", "spec")
        self.model = dict(doc.get("model", {}))
        self.hardware = dict(doc.get("hardware", {}))
        self.gp = dict(doc.get("gp", {}))
        devs = self.hardware.get("devices", [])
        self.G = int(sum(int(dv["count"]) for dv in devs))
        self._parse_features(doc.get("features"))
        self._parse_constraints(doc.get("constraints", []))
        # raw mixed radix: stride_{d-1} = 1, stride_j = stride_{j+1} * n_{j+1}
        d = len(self.features)
        self.strides = [1] * d
        for j in range(d - 2, -1, -1):
            self.strides[j] = self.strides[j + 1] * self.features[j + 1].n
        self.n_raw = self.strides[0] * self.features[0].n
        if self.n_raw > (1 << 63):
            raise SpaceError("schema", "raw index range exceeds 2^63")
        self._deps_init()
        if self.n_cvi() == 0:
            raise SpaceError("empty", "no configuration satisfies the constraints (S:34)")

    # ---------------------------------------------------------------- parsing / validation
    def _parse_features(self, feats):
        if not isinstance(feats, list) or len(feats) == 0:
            raise SpaceError("schema", "space must declare at least one feature (S:61)")
        names = [f.get("name") for f in feats]
        if len(set(names)) != len(names):
            raise SpaceError("schema", "feature names must be unique (S:34)")
        index = {nm: i for i, nm in enumerate(names)}
        # cycle detection first ("f1 references f2, f2 references f1 -> cyclic-dependency error")
        graph = {}
        for f in feats:
            refs = []
            for a in f.get("requires", []) or []:
                if a.get("feature") not in index:
                    raise SpaceError("unknown_ref", f"{f.get('name')} requires unknown feature {a.get('feature')}")
                refs.append(index[a["feature"]])
            graph[index[f["name"]]] = refs
        state = {}

        def dfs(u):
            state[u] = 1
            for v in graph[u]:
                if state.get(v) == 1:
                    raise SpaceError("cycle", f"activation cycle through {names[v]}")
                if state.get(v) is None:
                    dfs(v)
            state[u] = 2

        for u in graph:
            if state.get(u) is None:
                dfs(u)
        self.features = []
        for i, f in enumerate(feats):
            dom = f.get("domain")
            if not isinstance(dom, list) or len(dom) == 0:
                raise SpaceError("empty_domain", f"feature {f.get('name')} has an empty domain (S:58)")
            if f.get("kind") not in ("sparse", "dense"):
                raise SpaceError("schema", f"feature {f['name']}: kind must be sparse|dense")
            dflt = f.get("default", dom[0])
            matches = [k for k, v in enumerate(dom) if v == dflt and type(v) is type(dflt)]
            if not matches:
                raise SpaceError("schema", f"feature {f['name']}: default not in domain (S:30)")
            atoms = []
            for a in f.get("requires", []) or []:
                r = index[a["feature"]]
                if r >= i:
                    raise SpaceError("order", f"{f['name']} requires a later feature (S:30)")
                if a.get("op") not in OPS:
                    raise SpaceError("schema", f"bad op {a.get('op')}")
                atoms.append(Atom(r, a["op"], a["value"]))
            self.features.append(Feature(f["name"], f["kind"], list(dom), matches[0], atoms))
        self.index = index

    def _parse_constraints(self, cons):
        self.constraints = []
        for c in cons:
            t = c.get("type")
            refs = []
            if t in ("product_eq_devices", "product_le_devices_pow2", "divides_const", "gbs_divisible"):
                refs = [self._ref(n) for n in c["features"]]
            elif t == "divides":
                refs = [self._ref(c["a"]), self._ref(c["b"])]
            elif t == "seq_divisible_2cp":
                refs = [self._ref(c["feature"])]
            elif t == "ge":
                refs = [self._ref(c["a"]), self._ref(c["b"])]
            elif t == "le_const_div":
                refs = [self._ref(c["feature"])] + [self._ref(n) for n in c["div"]]
            elif t == "microbatch_divisible_pp":
                refs = [self._ref(c[k]) for k in ("vpp", "pp", "dp", "mbs")]
            elif t == "implies":
                refs = [self._ref(a["feature"]) for a in c["if"] + c["then"]]
            else:
                raise SpaceError("schema", f"unknown constraint type {t}")
            if t in ("divides_const", "le_const_div") and c["const"] not in self.model and c["const"] != "G":
                raise SpaceError("schema", f"unknown model constant {c['const']}")
            self.constraints.append((c, sorted(set(refs))))

    def _ref(self, name):
        if name not in self.index:
            raise SpaceError("unknown_ref", f"constraint references unknown feature {name}")
        return self.index[name]

    def const(self, name):
        return self.G if name == "G" else self.model[name]

    # ---------------------------------------------------------------- per-configuration rules
    def activity(self, digits):
        """active_j for every feature, in declaration order (SURVEY A.1 'Activity')."""
        act = []
        for f in self.features:
            ok = True
            for a in f.requires:
                if not act[a.ref] or not compare(self.features[a.ref].values[digits[a.ref]], a.op, a.value):
                    ok = False
                    break
            act.append(ok)
        return act

    def effective_value(self, j, digits, act):
        """Value used by constraints/simulator/GP: inactive -> default."""
        f = self.features[j]
        return f.values[digits[j] if act[j] else f.default_digit]

    def canonical(self, digits, act=None):
        """G1: every inactive feature carries its default digit."""
        act = self.activity(digits) if act is None else act
        return all(act[j] or digits[j] == f.default_digit for j, f in enumerate(self.features))

    def constraint_ok(self, c, digits, act):
        """One structural constraint, evaluated on effective values (reading R5)."""
        t = c["type"]
        ev = lambda name: _num(self.effective_value(self.index[name], digits, act))
        isact = lambda name: act[self.index[name]]
        if t == "product_eq_devices":
            return math.prod(ev(n) for n in c["features"]) == self.G
        if t == "product_le_devices_pow2":
            w = math.prod(ev(n) for n in c["features"])
            ok = w <= self.G and (w & (w - 1)) == 0
            if c.get("divides_devices", False):
                ok = ok and self.G % w == 0
            return ok
        if t == "divides":
            return ev(c["b"]) % ev(c["a"]) == 0
        if t == "divides_const":
            return self.const(c["const"]) % math.prod(ev(n) for n in c["features"]) == 0
        if t == "gbs_divisible":
            return self.model["GBS"] % math.prod(ev(n) for n in c["features"]) == 0
        if t == "seq_divisible_2cp":
            cp = ev(c["feature"])
            return cp == 1 or self.model["S"] % (2 * cp) == 0
        if t == "ge":
            if not (isact(c["a"]) and isact(c["b"])):
                return True
            return ev(c["a"]) >= ev(c["b"])
        if t == "le_const_div":
            if not isact(c["feature"]):
                return True
            return ev(c["feature"]) * math.prod(ev(n) for n in c["div"]) <= self.const(c["const"])
        if t == "microbatch_divisible_pp":
            if ev(c["vpp"]) <= 1:
                return True
            m = self.model["GBS"] // (ev(c["dp"]) * ev(c["mbs"]))
            return m % ev(c["pp"]) == 0
        if t == "implies":
            def atom(a):
                j = self.index[a["feature"]]
                return act[j] and compare(self.features[j].values[digits[j]], a["op"], a["value"])
            return (not all(atom(a) for a in c["if"])) or all(atom(a) for a in c["then"])
        raise SpaceError("schema", t)

    def structurally_valid(self, digits):
        """G1 and all non-resource constraints: membership in the CVI."""
        act = self.activity(digits)
        if not self.canonical(digits, act):
            return False
        return all(self.constraint_ok(c, digits, act) for c, _ in self.constraints)

    # ---------------------------------------------------------------- raw <-> digits
    def decode_raw(self, raw):
        """Digits by repeated div/mod, most significant first."""
        digits = []
        for j in range(len(self.features)):
            digits.append((raw // self.strides[j]) % self.features[j].n)
        return digits

    def encode_raw(self, digits):
        return sum(dg * s for dg, s in zip(digits, self.strides))

    # ---------------------------------------------------------------- CVI dynamic program
    def _deps_init(self):
        """For the DP: which earlier features can still influence the validity of a suffix."""
        d = len(self.features)
        self._last_ref = []                   # constraint -> highest referenced feature index
        for c, refs in self.constraints:
            self._last_ref.append(max(refs))
        self._needed = []                     # needed[j]: features < j whose (digit, active) matter for j..d-1
        for j in range(d + 1):
            need = set()
            for k in range(j, d):
                for a in self.features[k].requires:
                    if a.ref < j:
                        need.add(a.ref)
            for (c, refs), last in zip(self.constraints, self._last_ref):
                if last >= j:
                    need.update(r for r in refs if r < j)
            self._needed.append(sorted(need))

    def _extend_ok(self, j, digits, act):
        """Feature j has just been assigned: check G1 for it and every constraint it completes."""
        if not act[j] and digits[j] != self.features[j].default_digit:
            return False
        for (c, refs), last in zip(self.constraints, self._last_ref):
            if last == j and not self.constraint_ok(c, digits, act):
                return False
        return True

    def _act_of(self, j, digits, act):
        f = self.features[j]
        for a in f.requires:
            if not act[a.ref] or not compare(self.features[a.ref].values[digits[a.ref]], a.op, a.value):
                return False
        return True

    @lru_cache(maxsize=None)
    def _count_key(self, j, key):
        # key = tuple of (feature index, digit, active) for the needed earlier features.
        d = len(self.features)
        if j == d:
            return 1
        digits = [0] * d
        act = [False] * d
        for (i, dg, ac) in key:
            digits[i] = dg
            act[i] = ac
        total = 0
        for v in range(self.features[j].n):
            digits[j] = v
            act[j] = self._act_of(j, digits, act)
            if not self._extend_ok(j, digits, act):
                continue
            total += self._count_key(j + 1, self._key(j + 1, digits, act))
        return total

    def _key(self, j, digits, act):
        return tuple((i, digits[i], act[i]) for i in self._needed[j])

    def count_completions(self, j, digits, act):
        """Number of CVI members whose first j digits equal digits[:j] (prefix assumed valid)."""
        return self._count_key(j, self._key(j, digits, act))

    def n_cvi(self):
        return self._count_key(0, ())

    def cvi_unrank(self, p):
        """The p-th structurally valid raw index in ascending raw order -> digits."""
        if not 0 <= p < self.n_cvi():
            raise IndexError(p)
        d = len(self.features)
        digits = [0] * d
        act = [False] * d
        for j in range(d):
            for v in range(self.features[j].n):
                digits[j] = v
                act[j] = self._act_of(j, digits, act)
                if not self._extend_ok(j, digits, act):
                    continue
                c = self._count_key(j + 1, self._key(j + 1, digits, act))
                if p < c:
                    break
                p -= c
            else:
                raise AssertionError("unrank fell off the domain")
        return digits

    def cvi_rank(self, digits):
        """Inverse of cvi_unrank for a structurally valid configuration."""
        d = len(self.features)
        dg = [0] * d
        act = [False] * d
        p = 0
        for j in range(d):
            for v in range(digits[j]):
                dg[j] = v
                act[j] = self._act_of(j, dg, act)
                if self._extend_ok(j, dg, act):
                    p += self._count_key(j + 1, self._key(j + 1, dg, act))
            dg[j] = digits[j]
            act[j] = self._act_of(j, dg, act)
            if not self._extend_ok(j, dg, act):
                raise ValueError("configuration is not structurally valid")
        return p

    # ---- optimizer-driven batches
    def subtree_range(self, prefix):
        """MCTS subtree as a CVI range ("each node corresponds to a partial
        configuration ... each edge represents a valid refinement"): the members whose first
        len(prefix) digits equal `prefix` are the positions [begin, begin + count) -- contiguous
        because the CVI is ascending raw order with the first-declared feature most significant
        (R2, R4).  begin = members below the prefix, counted by the same prefix walk
        as cvi_rank; count = completions of the prefix (0 if the prefix itself is invalid)."""
        n = len(prefix)
        d = len(self.features)
        dg = [0] * d
        act = [False] * d
        p = 0
        for j in range(n):
            for v in range(prefix[j]):
                dg[j] = v
                act[j] = self._act_of(j, dg, act)
                if self._extend_ok(j, dg, act):
                    p += self._count_key(j + 1, self._key(j + 1, dg, act))
            dg[j] = prefix[j]
            act[j] = self._act_of(j, dg, act)
            if not self._extend_ok(j, dg, act):
                return p, 0
        return p, self._count_key(n, self._key(n, dg, act))

    def coordinate_neighbors(self, digits):
        """Coordinate-search candidates of a configuration ("perturbs the active parameter
        along its current search direction"; S:230-247 propose/update with step doubling), all
        at once (reading R19): for every ACTIVE dense feature in declaration order, every step
        2^e < n_f, direction +1 then -1, the configuration with that digit moved, if inside the
        domain and structurally valid (G1-G3)."""
        act = self.activity(digits)
        out = []
        for f, feat in enumerate(self.features):
            if feat.kind != "dense" or not act[f]:
                continue
            step = 1
            while step < feat.n:
                for sgn in (1, -1):
                    nd = digits[f] + sgn * step
                    if 0 <= nd < feat.n:
                        y = list(digits)
                        y[f] = nd
                        if self.structurally_valid(y):
                            out.append(y)
                step *= 2
        return out

    def enumerate_cvi(self):
        """Every structurally valid configuration exactly once, ascending raw."""
        d = len(self.features)
        digits = [0] * d
        act = [False] * d

        def rec(j):
            if j == d:
                yield list(digits)
                return
            for v in range(self.features[j].n):
                digits[j] = v
                act[j] = self._act_of(j, digits, act)
                if self._extend_ok(j, digits, act):
                    yield from rec(j + 1)

        yield from rec(0)


def load_space(text_or_path) -> Space:
    """Parse + validate a space JSON document (S:54-62 load_space)."""
    if isinstance(text_or_path, dict):
        return Space(text_or_path)
    s = str(text_or_path)
    if s.lstrip().startswith("{"):
        return Space(json.loads(s))
    with open(s) as fh:
        return Space(json.load(fh))
