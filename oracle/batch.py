"""Oracle, batch form: the same definitions as space.py / feistel.py / sim.py / gp.py, evaluated
over numpy arrays of candidates so that full-size workloads (C4's 10^8 samples, C5's whole
space) finish in minutes on the host cores.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Nothing here is a new algorithm; each function is the array form of a scalar oracle function,
pinned against it element by element in tests/test_oracle_batch.py:

  * Feistel.__call__  -> feistel_batch  (R3: same rounds, same keys, uint64 lanes; the
                                         cycle-walk repeats the permutation on the lanes still
                                         outside [0, n))
  * Space.cvi_unrank  -> Unranker.unrank (the memoised completion-count DP of space.py, written
                                         out as a table per feature: state = the DP key
                                         (needed earlier (digit, active) pairs), transition on
                                         digit v, count of completions of the next state; the
                                         digit loop "skip invalid v, break at p < c, else
                                         p -= c" becomes a cumulative-sum search over v)
  * sim.knob_arrays   -> knob_arrays    (effective value = value of the digit if active, else
                                         of the default digit, reading R5)
  * gp.features       -> features       (phi = digit_eff / (n - 1), x~ = phi / l; R9)
  * gp.cross_cov      -> cross_cov      (r = ||x~ - o~||_2 by direct differences, accumulated
                                         feature by feature; no ||x||^2 + ||o||^2 - 2 x.o)
"""

from __future__ import annotations

import numpy as np

from . import gp as _gp
from . import sim as _sim
from .feistel import Feistel

M32 = np.uint64(0xFFFFFFFF)


# ---------------------------------------------------------------- a0: SAMPLE permutation (R3)
def _fmix32(h):
    h = h & M32
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x85EBCA6B)) & M32
    h ^= h >> np.uint64(13)
    h = (h * np.uint64(0xC2B2AE35)) & M32
    h ^= h >> np.uint64(16)
    return h


def _E(x, a, c, keys):
    L, R = x >> np.uint64(c), x & np.uint64((1 << c) - 1)
    for k in keys:
        L, R = R, L ^ (_fmix32(R ^ np.uint64(k)) & np.uint64((1 << a) - 1))
        a, c = c, a
    return (L << np.uint64(c)) | R


def feistel_batch(n, seed, ordinals):
    """pi_seed(j) for an array of ordinals j in [0, n) (oracle/feistel.py, reading R3)."""
    f = Feistel(n, seed)
    j = np.asarray(ordinals, dtype=np.uint64)
    if j.size and int(j.max()) >= n:
        raise IndexError("ordinal outside [0, n)")
    x = _E(j, f.a, f.c, f.keys)
    out = x >= np.uint64(n)
    while out.any():
        x[out] = _E(x[out], f.a, f.c, f.keys)
        out = x >= np.uint64(n)
    return x.astype(np.int64)


# ---------------------------------------------------------------- a1: CVI unrank (R4)
class Unranker:
    """space.cvi_unrank over arrays.  Per feature j: the DP keys reachable at j (states), and for
    every (state, digit v): the activity of feature j, whether the extension is valid
    (space._extend_ok), the next state and its completion count (space._count_key)."""

    def __init__(self, space):
        self.space = space
        d = len(space.features)
        self.d = d
        self.trans, self.act, self.cnt = [], [], []
        keys = [()]                                    # states of level 0
        for j in range(d):
            n = space.features[j].n
            nxt_id = {}
            T = np.full((len(keys), n), -1, dtype=np.int64)
            A = np.zeros((len(keys), n), dtype=bool)
            C = np.zeros((len(keys), n), dtype=np.int64)
            for s, key in enumerate(keys):
                digits = [0] * d
                act = [False] * d
                for (i, dg, ac) in key:
                    digits[i] = dg
                    act[i] = ac
                for v in range(n):
                    digits[j] = v
                    act[j] = space._act_of(j, digits, act)
                    A[s, v] = act[j]
                    if not space._extend_ok(j, digits, act):
                        continue
                    k2 = space._key(j + 1, digits, act)
                    if k2 not in nxt_id:
                        nxt_id[k2] = len(nxt_id)
                    T[s, v] = nxt_id[k2]
                    C[s, v] = space._count_key(j + 1, k2)
            self.trans.append(T)
            self.act.append(A)
            self.cnt.append(C)
            keys = sorted(nxt_id, key=nxt_id.get)
        self.strides = np.array(space.strides, dtype=np.int64)
        self.n_cvi = space.n_cvi()

    def unrank(self, p):
        """CVI positions -> (digits [B, d] int64, active [B, d] bool, raw [B] int64)."""
        p = np.array(p, dtype=np.int64, copy=True)
        if p.size and (p.min() < 0 or p.max() >= self.n_cvi):
            raise IndexError("CVI position outside [0, n_cvi)")
        B = p.size
        digits = np.zeros((B, self.d), dtype=np.int64)
        active = np.zeros((B, self.d), dtype=bool)
        s = np.zeros(B, dtype=np.int64)
        rows = np.arange(B)
        for j in range(self.d):
            C = self.cnt[j]                             # 0 for invalid extensions
            cum = np.cumsum(C, axis=1)                  # [states, n]
            cs = cum[s]                                 # [B, n]
            v = np.sum(p[:, None] >= cs, axis=1)        # first digit with p < cumulative count
            p -= cs[rows, v] - C[s, v]
            digits[:, j] = v
            active[:, j] = self.act[j][s, v]
            s = self.trans[j][s, v]
        assert (s >= 0).all()
        return digits, active, digits @ self.strides


# ---------------------------------------------------------------- a3 inputs / a4 features
def _knob_value(k, v):
    if k == "ar":
        return float(_sim._ar_code(v))
    if k == "disp":
        return 1.0 if v == "allgather" else 0.0
    if isinstance(v, bool):
        return 1.0 if v else 0.0
    return float(v)


def effective_digits(space, digits, active):
    dflt = np.array([f.default_digit for f in space.features], dtype=np.int64)
    return np.where(active, digits, dflt[None, :])


def knob_arrays(space, digits, active):
    """sim.knob_arrays over arrays of digits / activity."""
    names = _sim.TRAIN_KNOBS if space.sim_mode in ("spec", "derived") else _sim.SERVE_KNOBS
    B = digits.shape[0]
    eff = effective_digits(space, digits, active)
    vals, acts, present = {}, {}, {}
    for k in names:
        present[k] = k in space.index
        if present[k]:
            j = space.index[k]
            tab = np.array([_knob_value(k, v) for v in space.features[j].values], dtype=np.float64)
            vals[k] = tab[eff[:, j]]
            acts[k] = active[:, j].copy()
        else:
            vals[k] = np.full(B, _knob_value(k, _sim.NEUTRAL[k]), dtype=np.float64)
            acts[k] = np.zeros(B, dtype=bool)
    return vals, acts, present


def simulate(space, digits, active, terms=False):
    return _sim.simulate_knobs(space, *knob_arrays(space, digits, active), terms=terms)


def features(space, digits, active):
    """gp.features over arrays: x~_j = (digit_eff_j / (n_j - 1)) / l_j (0 if n_j == 1)."""
    ls = _gp.lengthscales(space)
    eff = effective_digits(space, digits, active).astype(np.float64)
    den = np.array([f.n - 1 if f.n > 1 else 1 for f in space.features], dtype=np.float64)
    one = np.array([f.n > 1 for f in space.features])
    phi = np.where(one[None, :], eff / den[None, :], 0.0)
    return phi / ls[None, :]


def cross_cov(space, X, O):
    """gp.cross_cov with r^2 accumulated one feature at a time (direct differences)."""
    r2 = np.zeros((X.shape[0], O.shape[0]), dtype=np.float64)
    for j in range(X.shape[1]):
        dj = X[:, j, None] - O[None, :, j]
        r2 += dj * dj
    return _gp.kernel_r(space, np.sqrt(r2))


def posterior(fit, X, m0, Kinv=None):
    """Fit.posterior (mu = m0 + b + k*.alpha, s2 = max(sf2 - k*^T K^-1 k*, 0)) for a large batch;
    K^-1 k* by numpy.linalg.solve as in gp.Fit (or a precomputed K^-1 applied by one product)."""
    if fit.M == 0:
        return m0 + 0.0, np.full(len(m0), fit.sf2)
    ks = cross_cov(fit.space, X, fit.O)
    mu = m0 + fit.b + ks @ fit.alpha
    sol = np.linalg.solve(fit.K, ks.T) if Kinv is None else Kinv @ ks.T
    s2 = np.maximum(fit.sf2 - np.sum(ks.T * sol, axis=0), 0.0)
    return mu, s2
