"""Brute-force enumeration over the FULL raw index range -- the independent pin for the
oracle's memoised CVI dynamic program (tests only).

Every raw index 0..N_raw-1 is decoded by div/mod, then gate activity,
canonical-inactive G1 (S:29 default), and each structural constraint of the preset are
evaluated exhaustively with numpy.  No pruning, no memoisation, no per-structure tables.
"""

import math

import numpy as np


def _numeric(v):
    if isinstance(v, bool):
        return 1.0 if v else 0.0
    if isinstance(v, str):
        return float("nan")
    return float(v)


def _cmp(a, op, b):
    return {">": a > b, ">=": a >= b, "==": a == b, "!=": a != b, "<": a < b, "<=": a <= b}[op]


def enumerate_valid_raw(doc, G, chunk=1 << 22, window=None):
    """-> sorted np.ndarray of raw indices (optionally within window=(lo, hi)) satisfying G1 and every
    structural constraint."""
    feats = doc["features"]
    names = [f["name"] for f in feats]
    idx = {n: i for i, n in enumerate(names)}
    sizes = [len(f["domain"]) for f in feats]
    d = len(feats)
    strides = [1] * d
    for j in range(d - 2, -1, -1):
        strides[j] = strides[j + 1] * sizes[j + 1]
    n_raw = strides[0] * sizes[0]
    vals = [np.array([_numeric(v) for v in f["domain"]]) for f in feats]
    dflt = [next(i for i, v in enumerate(f["domain"]) if v == f.get("default", f["domain"][0])
                 and type(v) is type(f.get("default", f["domain"][0]))) for f in feats]
    model = doc.get("model", {})
    const = lambda n: G if n == "G" else model[n]
    out = []
    w_lo, w_hi = window if window is not None else (0, n_raw)
    for lo in range(w_lo, w_hi, chunk):
        raw = np.arange(lo, min(w_hi, lo + chunk), dtype=np.int64)
        D = [(raw // strides[j]) % sizes[j] for j in range(d)]
        act = []
        for j, f in enumerate(feats):
            a = np.ones(len(raw), dtype=bool)
            for at in f.get("requires", []) or []:
                r = idx[at["feature"]]
                dom = feats[r]["domain"]
                allowed = np.array([bool(_cmp(v, at["op"], at["value"])) if not isinstance(v, str) or at["op"] in ("==", "!=")
                                    else False for v in dom])
                a &= act[r] & allowed[D[r]]
            act.append(a)
        ok = np.ones(len(raw), dtype=bool)
        for j in range(d):
            ok &= act[j] | (D[j] == dflt[j])
        eff = lambda n: np.where(act[idx[n]], vals[idx[n]][D[idx[n]]], vals[idx[n]][dflt[idx[n]]])
        for c in doc.get("constraints", []):
            t = c["type"]
            if t == "product_eq_devices":
                ok &= math.prod(eff(n) for n in c["features"]) == G
            elif t == "product_le_devices_pow2":
                w = math.prod(eff(n) for n in c["features"]).astype(np.int64)
                cc = (w <= G) & ((w & (w - 1)) == 0)
                if c.get("divides_devices"):
                    cc &= (G % w) == 0
                ok &= cc
            elif t == "divides":
                ok &= np.mod(eff(c["b"]), eff(c["a"])) == 0
            elif t == "divides_const":
                ok &= np.mod(const(c["const"]), math.prod(eff(n) for n in c["features"])) == 0
            elif t == "gbs_divisible":
                ok &= np.mod(model["GBS"], math.prod(eff(n) for n in c["features"])) == 0
            elif t == "seq_divisible_2cp":
                cp = eff(c["feature"])
                ok &= (cp == 1) | (np.mod(model["S"], 2 * cp) == 0)
            elif t == "ge":
                both = act[idx[c["a"]]] & act[idx[c["b"]]]
                ok &= ~both | (eff(c["a"]) >= eff(c["b"]))
            elif t == "le_const_div":
                a = act[idx[c["feature"]]]
                ok &= ~a | (eff(c["feature"]) * math.prod(eff(n) for n in c["div"]) <= const(c["const"]))
            elif t == "microbatch_divisible_pp":
                vpp = eff(c["vpp"])
                m = model["GBS"] // (eff(c["dp"]) * eff(c["mbs"]))
                ok &= (vpp <= 1) | (np.mod(m, eff(c["pp"])) == 0)
            elif t == "implies":
                def atom(a):
                    r = idx[a["feature"]]
                    dom = feats[r]["domain"]
                    allowed = np.array([bool(_cmp(v, a["op"], a["value"])) for v in dom])
                    return act[r] & allowed[D[r]]
                cond = np.ones(len(raw), dtype=bool)
                for a in c["if"]:
                    cond &= atom(a)
                then = np.ones(len(raw), dtype=bool)
                for a in c["then"]:
                    then &= atom(a)
                ok &= ~cond | then
            else:
                raise ValueError(t)
        out.append(raw[ok])
    return np.concatenate(out)
