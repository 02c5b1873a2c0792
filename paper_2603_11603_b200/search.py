"""Algorithm 1: the AutoScout search loop over the library.

The loop itself is sequential control (one 2x2 batch per iteration); it runs on the host and calls
the C-ABI library for everything data-parallel or exact: configuration decode / validity /
simulator (autoscout_simulate, the low-fidelity evaluation), subtree ranges of partial sparse
assignments (autoscout_subtree_range, MCTS rollouts), and -- at the fidelity switch -- the
certified top-K of the whole space under the simulator (score_batch + topk, the hot path), which
is "the top-K configurations identified during simulation ... prioritized for re-evaluation under
real profiling" at the scale the GPU makes possible.

Components, each after the passage it implements; the paper leaves the formulas to the reader,
SPEC.md fixes them and every SPEC reading is listed in DESIGN.md (R22):
  * UCB1 arm choice, Eq. 1: a_t = argmax_a Q_a/N_a + C(t) sqrt(ln N_total / N_a),
    C(t) = C0 gamma^t; unpulled arms first, ties -> Sparse.
  * difference-of-differences reward of the 2x2 batch:
    D_sparse = ((c_bb - c_cb) + (c_bc - c_cc)) / 2, D_dense = ((c_bb - c_bc) + (c_cb - c_cc)) / 2,
    bandit reward clip(D / c_bb, 0, 1).
  * tournament warm start over K feature orderings: zigzag
    order across rounds, one proposal per survivor per round, shared evaluation propagated to
    every tree, keep the top half by cumulative reward (ties -> lower index).
  * sparse optimizer: MCTS over the structural prefix features in the tree's ordering (PAPER.md:
    143-146): UCT (c_uct = 1.414, unvisited first), one expansion per proposal, random feasible
    completion (a uniform CVI position of the node's subtree), reward r = c_ref / c.
  * dense optimizer: coordinate search with step doubling on success, one direction flip then
    the next coordinate on failure, reflecting boundaries, projection onto the active features
    (SPEC.md:230-262).
  * fidelity-adaptive evaluation: simulated costs, real
    profiling of the best-simulated and the batch argmin every tau iterations, MAPE over the
    window, one-way switch when MAPE > epsilon: MCTS trees retained, bandit (Q, N) scaled by
    lambda (weak priors), the K_reval best configurations by simulated cost re-evaluated.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SPARSE, DENSE = 0, 1


# ---------------------------------------------------------------- bandit (Eq. 1)
def exploration(C0, gamma, t):
    """C(t) = C0 gamma^t."""
    return C0 * gamma ** t


def select_arm(Q, N, t, C0=1.414, gamma=0.995):
    """Eq. 1: argmax_a Q_a/N_a + C(t) sqrt(ln N_total / N_a); an unpulled arm first (Sparse before
    Dense), ties -> Sparse."""
    for a in (SPARSE, DENSE):
        if N[a] == 0:
            return a
    n_tot = N[SPARSE] + N[DENSE]
    c = exploration(C0, gamma, t)
    v = [Q[a] / N[a] + c * math.sqrt(math.log(n_tot) / N[a]) for a in (SPARSE, DENSE)]
    return SPARSE if v[SPARSE] >= v[DENSE] else DENSE


def attribute(c_bb, c_bc, c_cb, c_cc):
    """Difference-of-differences on the 2x2 batch (lower cost better) -> (D_sparse, D_dense,
    r_sparse, r_dense); rewards clip(D / c_bb, 0, 1), infinite (infeasible) cells count 0."""
    if not math.isfinite(c_bb):
        return 0.0, 0.0, 0.0, 0.0
    def half_sum(a, b):                     # an infeasible candidate cell: -inf, never nan
        v = 0.5 * (a + b)
        return -math.inf if math.isnan(v) else v
    d_s = half_sum(c_bb - c_cb, c_bc - c_cc)
    d_d = half_sum(c_bb - c_bc, c_cb - c_cc)
    clip = lambda d: min(1.0, max(0.0, d / c_bb)) if math.isfinite(d) else 0.0
    return d_s, d_d, clip(d_s), clip(d_d)


def mape(pairs):
    """Mean absolute percentage error of (predicted, real) pairs: mean |pred - real| / real
    (SPEC.md:418-421)."""
    return float(np.mean([abs(p - q) / q for p, q in pairs]))


def weak_prior(Q, N, lam):
    """Bandit statistics at the fidelity switch, "treated as weak priors rather than reset"
    (PAPER.md:264): both scaled by lam, so every Q_a / N_a is kept."""
    return [q * lam for q in Q], [n * lam for n in N]


# ---------------------------------------------------------------- tournament
@dataclass
class Tournament:
    """K candidate tree orderings; zigzag rounds; keep the top half."""
    K: int
    survivors: list = field(default_factory=list)
    reward: list = field(default_factory=list)
    round: int = 0
    pos: int = 0

    def __post_init__(self):
        self.survivors = list(range(self.K))
        self.reward = [0.0] * self.K

    @property
    def done(self):
        return len(self.survivors) <= 1

    def order(self):
        """This round's proposal order: ascending on even rounds, descending on odd ones."""
        return self.survivors if self.round % 2 == 0 else self.survivors[::-1]

    def next(self):
        return self.order()[self.pos]

    def record(self, proposer, r):
        """Add the proposer's reward; at the end of a round keep the top ceil(n/2) survivors by
        cumulative reward, ties -> lower original index."""
        self.reward[proposer] += r
        self.pos += 1
        if self.pos == len(self.survivors):
            keep = (len(self.survivors) + 1) // 2
            ranked = sorted(self.survivors, key=lambda i: (-self.reward[i], i))
            self.survivors = sorted(ranked[:keep])
            self.round += 1
            self.pos = 0

    def winner(self):
        return self.survivors[0]


# ---------------------------------------------------------------- MCTS over the structural prefix
class MctsTree:
    """Dependency-aware search tree over the structural features in `order` (a permutation of the
    structural prefix that respects gate ancestry); nodes keyed by the assigned (feature, digit)
    pairs.  Feasibility of a partial assignment = its subtree in the library's CVI is non-empty."""

    def __init__(self, space, order, c_uct=1.414, rng=None):
        self.sp = space
        self.order = list(order)
        self.c_uct = c_uct
        self.N = {(): 0}
        self.W = {(): 0.0}
        self.rng = rng or np.random.default_rng(0)

    def _digits_of(self, key):
        dg = {}
        for f, v in key:
            dg[f] = v
        return dg

    def _feasible_children(self, key):
        """Structural feature: digits whose structural subtree is non-empty.  Sparse tail feature:
        every digit, or only the default when its gate ancestors are all assigned and switch it
        off (constraints on tail digits are met by the completion)."""
        j = len(key)
        f = self.order[j]
        part = self._digits_of(key)
        out = []
        if f < self.sp.n_prefix:
            for v in range(self.sp.nvals[f]):
                if self.sp.structure_count({**part, f: v}) > 0:
                    out.append(key + ((f, v),))
            return out
        if self.sp.gated_off(part, f):
            return [key + ((f, self.sp.dflt[f]),)]
        return [key + ((f, v),) for v in range(self.sp.nvals[f])]

    def propose(self, explore=True):
        """UCT descent (unvisited children first, a seeded random one), one expansion, random
        feasible completion -> full raw index.  explore=False: greedy descent (c_uct = 0) through
        visited children -- the non-selected arm's exploitation move."""
        key = ()
        c_uct = self.c_uct if explore else 0.0
        while len(key) < len(self.order):
            kids = self._feasible_children(key)
            if not kids:
                break
            unvisited = [k for k in kids if self.N.get(k, 0) == 0]
            if unvisited and (explore or len(unvisited) == len(kids)):
                key = unvisited[int(self.rng.integers(len(unvisited)))]
                self.N.setdefault(key, 0)
                self.W.setdefault(key, 0.0)
                break
            lnp = math.log(max(self.N[key], 1))
            seen = [k for k in kids if self.N.get(k, 0) > 0]
            key = max(seen, key=lambda k: (self.W[k] / self.N[k] + c_uct * math.sqrt(lnp / self.N[k]),
                                           -kids.index(k)))
        return self.sp.complete(self._digits_of(key), self.rng)

    def backpropagate(self, raw, r):
        """Root-to-leaf path of the configuration's structural digits under this ordering (created
        if absent): N += 1, W += r on every node ("for backpropagation")."""
        dg = self.sp.digits(raw)
        key = ()
        self.N[key] = self.N.get(key, 0) + 1
        self.W[key] = self.W.get(key, 0.0) + r
        for f in self.order:
            key = key + ((f, dg[f]),)
            self.N[key] = self.N.get(key, 0) + 1
            self.W[key] = self.W.get(key, 0.0) + r

    def n_nodes(self):
        return len(self.N)


# ---------------------------------------------------------------- dense coordinate search
@dataclass
class DenseState:
    """Coordinate-wise search over the active dense features."""
    coord: int = 0
    direction: dict = field(default_factory=dict)
    step: dict = field(default_factory=dict)
    flip_used: bool = False
    step_cap: int = 8

    def propose(self, sp, raw, explore=True):
        """The active coordinate moved by its step in its direction (reflected at the grid ends);
        explore=False: a single grid step (the non-selected arm's local move).
        -> raw (unchanged when the configuration has no active dense feature)."""
        act = sp.active_dense(raw)
        if not act:
            return raw
        f = act[self.coord % len(act)]
        dg = sp.digits(raw)
        d = self.direction.get(f, 1)
        s = self.step.get(f, 1) if explore else 1
        n = sp.nvals[f]
        nd = dg[f] + d * s
        if not 0 <= nd < n:
            d = -d
            self.direction[f] = d
            nd = min(max(dg[f] + d * s, 0), n - 1)
        dg[f] = nd
        return sp.valid_raw(dg, raw)

    def update(self, sp, raw, improved):
        act = sp.active_dense(raw)
        if not act:
            return
        f = act[self.coord % len(act)]
        if improved:
            self.step[f] = min(2 * self.step.get(f, 1), self.step_cap)
            self.flip_used = False
        else:
            self.step[f] = 1
            if not self.flip_used:
                self.direction[f] = -self.direction.get(f, 1)
                self.flip_used = True
            else:
                self.coord = (self.coord + 1) % len(act)
                self.flip_used = False


# ---------------------------------------------------------------- the space adapter
class SearchSpace:
    """Host view of a library handle for the loop: digits, activity, feasibility counts and
    completions through the C ABI (no decode logic here)."""

    def __init__(self, lib_space):
        self.L = lib_space
        feats = lib_space.doc["features"]
        self.names = [f["name"] for f in feats]
        self.nvals = [len(f["domain"]) for f in feats]
        self.dense = [f.get("kind") == "dense" for f in feats]
        self.d = len(feats)
        self.n_prefix = lib_space.space_info()["n_prefix"]
        self.dflt = [f["domain"].index(f.get("default", f["domain"][0])) for f in feats]
        idx = {n: i for i, n in enumerate(self.names)}
        self.gates = [sorted({idx[a["feature"]] for a in (f.get("requires") or [])}) for f in feats]
        self.sparse = [f for f in range(self.d) if not self.dense[f]]

    def digits(self, raw):
        return list(self.L.decode(int(raw))[0])

    def ancestors(self, f):
        out, stack = set(), list(self.gates[f])
        while stack:
            g = stack.pop()
            if g not in out:
                out.add(g)
                stack.extend(self.gates[g])
        return out

    def gated_off(self, partial, f):
        """True if every gate ancestor of f is assigned in `partial` and f is inactive there."""
        anc = self.ancestors(f)
        if not anc or not anc <= set(partial):
            return False
        dg = list(self.dflt)
        for g, v in partial.items():
            dg[g] = v
        return not self.L.activity(self.raw_of(dg))[f]

    def project(self, dg):
        """Inactive features -> default digit (iterated: activity depends on earlier digits)."""
        dg = list(dg)
        for _ in range(self.d):
            act = self.L.activity(self.raw_of(dg))
            nd = [v if act[f] else self.dflt[f] for f, v in enumerate(dg)]
            if nd == dg:
                break
            dg = nd
        return dg

    def structure_count(self, partial):
        """Members whose structural digits extend `partial` ({feature: digit}; tail entries are
        ignored): subtree counts of the declaration-order prefix, summed over the unassigned
        earlier structural features."""
        partial = {f: v for f, v in partial.items() if f < self.n_prefix}
        fixed = sorted(partial)
        last = max(fixed) if fixed else -1
        total = 0
        for prefix in self._prefixes(partial, last + 1):
            total += self.L.subtree_range(prefix)[1]
        return total

    def _prefixes(self, partial, upto):
        out = [[]]
        for f in range(upto):
            vals = [partial[f]] if f in partial else range(self.nvals[f])
            out = [p + [v] for p in out for v in vals]
            if len(out) > 4096:
                raise ValueError("partial assignment too sparse to enumerate")
        return out

    def complete(self, partial, rng, tries=20):
        """A random CVI member extending `partial`: a uniform member of the structural subtree
        with the assigned tail digits written over it and projected onto the active features;
        retried while that violates a constraint, else the member itself -> raw."""
        tail = {f: v for f, v in partial.items() if f >= self.n_prefix}
        for _ in range(tries if tail else 1):
            raw = self._complete_structural(partial, rng)
            if not tail:
                return raw
            dg = self.digits(raw)
            for f, v in tail.items():
                dg[f] = v
            dg = self.project(dg)
            if self.L.raw_to_cvi(self.raw_of(dg))[1]:
                return self.raw_of(dg)
        return raw

    def _complete_structural(self, partial, rng):
        partial = {f: v for f, v in partial.items() if f < self.n_prefix}
        ranges = [self.L.subtree_range(p) for p in self._prefixes(partial, (max(partial) + 1) if partial else 0)]
        sizes = np.array([c for _, c in ranges], dtype=np.float64)
        if sizes.sum() == 0:
            raise ValueError("infeasible partial assignment")
        i = int(rng.choice(len(ranges), p=sizes / sizes.sum()))
        b, c = ranges[i]
        return int(self.L.cvi_to_raw(b + int(rng.integers(c))))

    def active_dense(self, raw):
        """Dense features active in this configuration, declaration order (PAPER.md:171 M(s))."""
        act = self.L.activity(int(raw))
        return [f for f in range(self.d) if self.dense[f] and act[f]]

    def raw_of(self, dg):
        return sum(int(v) * int(s) for v, s in zip(dg, self.strides()))

    def valid_raw(self, dg, fallback):
        raw = self.raw_of(dg)
        _, member = self.L.raw_to_cvi(raw)
        return raw if member else fallback

    def strides(self):
        s = [1] * self.d
        for j in range(self.d - 2, -1, -1):
            s[j] = s[j + 1] * self.nvals[j + 1]
        return s

    def swap_structure(self, raw_s, raw_x):
        """(S from raw_s, X from raw_x): the structural digits of raw_s with raw_x's tail digits
        projected onto the features active under S -- an inactive feature takes its default digit
        ("projects its current state onto X(s) by masking inactive dimensions").  If
        the projection violates a constraint, S keeps its own tail (raw_s)."""
        ds, dx = self.digits(raw_s), self.digits(raw_x)
        # S = its sparse digits (structural prefix and sparse tail), X = the dense digits
        dg = [ds[f] if (f < self.n_prefix or not self.dense[f]) else dx[f] for f in range(self.d)]
        return self.valid_raw(self.project(dg), int(raw_s))


# ---------------------------------------------------------------- Algorithm 1
@dataclass
class RunConfig:
    T: int = 50
    tau: int = 5
    epsilon: float = 0.1
    C0: float = 1.414
    gamma: float = 0.995
    c_uct: float = 1.414
    K: int = 4
    K_reval: int = 5
    lam: float = 0.25
    seed: int = 0
    gpu_topk: bool = True       # re-evaluation queue from the library's certified top-K of the space


def run(lib_space, real_cost, cfg: RunConfig, orderings=None, sim_cost=None):
    """Algorithm 1.  real_cost(raw) -> cost (profiling; here synthetic truth), sim_cost(raw) ->
    cost (default: the library's analytical simulator).  -> dict(best_raw, best_cost, trace, ...)."""
    sp = SearchSpace(lib_space)
    rng = np.random.default_rng(cfg.seed)
    sim_cost = sim_cost or (lambda r: lib_space.simulate(r)[0])
    if orderings is None:
        base = list(sp.sparse)
        orderings = [base, base[::-1]] + [list(rng.permutation(base)) for _ in range(max(0, cfg.K - 2))]
    orderings = [o for o in orderings[:cfg.K]]
    trees = [MctsTree(sp, o, cfg.c_uct, np.random.default_rng(cfg.seed * 7919 + i)) for i, o in enumerate(orderings)]
    mode = "sim"
    cache = {}                     # raw -> (cost, fidelity)
    counts = {"sim": 0, "real": 0}
    window = []                    # (predicted, real) pairs since the last checkpoint
    trace = []

    def evaluate(raw, force_real=False):
        raw = int(raw)
        hit = cache.get(raw)
        if hit is not None and (hit[1] == "real" or (mode == "sim" and not force_real)):
            return hit[0]
        if mode == "real" or force_real:
            c = real_cost(raw)
            counts["real"] += 1
            cache[raw] = (c, "real")
        else:
            c = sim_cost(raw)
            counts["sim"] += 1
            cache[raw] = (c, "sim")
        return c

    c_ref = None

    def reward(c):
        return c_ref / c if (c_ref is not None and math.isfinite(c) and c > 0) else 0.0

    # Phase 0: tournament warm start (Alg. 1 line 5)
    tour = Tournament(len(trees))
    while not tour.done:
        k = tour.next()
        raw = trees[k].propose()
        c = evaluate(raw)
        if c_ref is None:
            c_ref = c
        r = reward(c)
        for tr in trees:                      # shared learning: one evaluation, every tree
            tr.backpropagate(raw, r)
        tour.record(k, r)
    tree = trees[tour.winner()]

    def fresh_structure(s_from, explore=True, tries=8):
        """A sparse candidate whose structure differs from s_from's (a 2x2 batch with equal sparse
        cells measures nothing about the sparse arm); exploring proposals after a greedy miss."""
        key = lambda r: [sp.digits(r)[f] for f in sp.sparse]
        base = key(s_from)
        cand = tree.propose(explore=explore)
        for _ in range(tries):
            if key(cand) != base:
                break
            cand = tree.propose(explore=True)
        return cand

    # Phase 1 (lines 7-12)
    Q, N = [0.0, 0.0], [0, 0]
    dense = DenseState()
    s_base = tree.propose()
    s_cand = fresh_structure(s_base)
    x_base = s_base
    x_cand = dense.propose(sp, x_base)
    if c_ref is None:
        c_ref = evaluate(s_base)
    best = (s_base, evaluate(s_base))

    # Phase 2 (lines 14-29)
    for t in range(1, cfg.T + 1):
        cells = [sp.swap_structure(s, x) for s in (s_base, s_cand) for x in (x_base, x_cand)]
        c = [evaluate(r) for r in cells]                                 # C_bb, C_bc, C_cb, C_cc
        # periodic validation + one-way fidelity switch (lines 20-21)
        if mode == "sim" and t % cfg.tau == 0:
            sims = [(v[0], r) for r, v in cache.items() if v[1] == "sim"]
            check = {min(sims)[1], cells[int(np.argmin(c))]} if sims else {cells[int(np.argmin(c))]}
            for r in check:
                pred = sim_cost(r)
                window.append((pred, evaluate(r, force_real=True)))
            err = mape(window)
            window.clear()
            if err > cfg.epsilon:
                mode = "real"
                nodes_at_switch = tree.n_nodes()
                Q, N = weak_prior(Q, N, cfg.lam)
                queue = sorted({r for r, v in cache.items() if v[1] == "sim"}, key=lambda r: cache[r][0])
                if cfg.gpu_topk:
                    queue = _library_topk(lib_space, cfg.K_reval) + queue
                seen = []
                for r in queue:
                    if r not in seen:
                        seen.append(r)
                    if len(seen) == cfg.K_reval:
                        break
                for r in seen:
                    cr = evaluate(r)
                    if cr < best[1]:
                        best = (r, cr)
                trace.append(dict(t=t, event="switch", mape=err, reval=seen, tree_nodes=nodes_at_switch,
                                  tree_nodes_after=tree.n_nodes()))
                c = [evaluate(r) for r in cells]
        # UpdateBest (line 23); a best found in simulation is re-validated on the real oracle
        i = int(np.argmin(c))
        if c[i] < best[1] or (mode == "real" and cache.get(best[0], (0, "sim"))[1] == "sim"):
            best = (cells[i], c[i]) if c[i] < evaluate(best[0]) else (best[0], evaluate(best[0]))
        d_s, d_d, r_s, r_d = attribute(*c)
        a = select_arm(Q, N, t, cfg.C0, cfg.gamma)
        Q[SPARSE] += r_s
        Q[DENSE] += r_d
        N[a] += 1
        for r, cc in zip(cells, c):
            tree.backpropagate(r, reward(cc))
        trace.append(dict(t=t, arm=a, mode=mode, c=c, d_sparse=d_s, d_dense=d_d, best=best[1]))
        # next pairs (lines 27-28): bases advance to the batch-argmin components; the selected arm
        # proposes a fresh candidate, the other keeps an improving candidate or regenerates
        bi = int(np.argmin(c))
        improved_d = min(c[1], c[3]) < min(c[0], c[2])
        dense.update(sp, x_base, improved_d)
        s_base = (s_base, s_cand)[bi // 2]
        x_base = (x_base, x_cand)[bi % 2]
        # both candidates are fresh every iteration (an improving candidate became the base); the
        # arm chosen by Eq. 1 explores (UCT / momentum step), the other exploits (greedy / one step)
        s_cand = fresh_structure(s_base, explore=(a == SPARSE))
        x_cand = dense.propose(sp, x_base, explore=(a == DENSE))
    if cache.get(best[0], (0, "sim"))[1] == "sim":       # the reported best is a real measurement
        best = (best[0], evaluate(best[0], force_real=True))
    return dict(best_raw=best[0], best_cost=best[1], trace=trace, real_evals=counts["real"],
                sim_evals=counts["sim"], mode=mode, tree_nodes=tree.n_nodes(), bandit=(Q, N),
                tournament_rounds=tour.round, winner=tour.winner())


def _library_topk(lib_space, k):
    """The K best configurations of the whole space under the simulator (acquisition SIM), certified
    top-K from the GPU scoring path -> raws ("top-K ... prioritized for re-evaluation")."""
    n = lib_space.n_cvi
    lib_space.score_batch(mode="range", begin=0, count=n, acq="sim", k=max(k, 1))
    return [r for r, _ in lib_space.topk(max(k, 1))]
