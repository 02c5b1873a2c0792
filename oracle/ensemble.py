"""Oracle: the paper's regression-simulator ensemble as the GP prior mean.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md Appendix B and SPEC.md fit_simulator / ensemble_predict:
  * four linear-regression simulators on the knob subsets of Table 2:
      3D-Parallelism      a100, a40, mbs, tp, pp, dp
      5D-Parallelism      a100, a40, mbs, tp, pp, dp, ep, cp, sp
      DDP-Aware           a100, a40, mbs, tp, pp, dp, ddp_optim
      Communication-Aware a100, a40, mbs, tp, pp, dp, ar, tp_comm
    (knobs that are not features of the space are dropped; ddp_optim is the feature "dopt",
    else "ddp" -- DESIGN.md reading R20);
  * numeric encoding of a knob = the value of its digit, inactive knobs at their default
    ("inactive features encoded as their default value"; G1 puts the default digit there);
  * fit on the seeded 80 % training part, R^2 on the 20 % holdout;
  * weights w_i = max(0, R^2_i) / sum_j max(0, R^2_j); all R^2 <= 0 -> Unavailable (P:546-548,
    S:406-408), and the prior falls back to the analytical simulator (reading R20).
Readings (R20): the regression target is y = ln c (the GP's own target, R9); the
"ridge fallback with penalty 1e-6" is applied to every fit on standardised columns
(intercept unpenalised), which equals OLS to ~1e-6 relative when the design is well posed and
keeps rank-deficient designs (few observations, collinear knobs) deterministic; holdout =
the floor(n/5) (at least 1) observations with the smallest splitmix64(seed ^ 0xE45E ^ i); a model
needs |train| >= p + 2 ("pre: >= |subset|+2 samples"), else it is unavailable.
"""

from __future__ import annotations

import numpy as np

from .feistel import splitmix64

TABLE2 = [
    ("3D-Parallelism", ["a100", "a40", "mbs", "tp", "pp", "dp"]),
    ("5D-Parallelism", ["a100", "a40", "mbs", "tp", "pp", "dp", "ep", "cp", "sp"]),
    ("DDP-Aware", ["a100", "a40", "mbs", "tp", "pp", "dp", "ddp_optim"]),
    ("Communication-Aware", ["a100", "a40", "mbs", "tp", "pp", "dp", "ar", "tp_comm"]),
]
RIDGE = 1e-6


def subset_features(space, knobs):
    """Table 2 knob names -> feature indices of this space (declaration order)."""
    names = [f.name for f in space.features]
    out = []
    for k in knobs:
        cands = ["dopt", "ddp"] if k == "ddp_optim" else [k]
        for c in cands:
            if c in names:
                out.append(names.index(c))
                break
    return sorted(set(out))


def encode(space, digits, cols):
    """Numeric encodings of the knobs `cols` (value of the digit; inactive knobs carry the default)."""
    return np.array([[float(space.features[j].numeric(dg[j])) for j in cols] for dg in digits], dtype=np.float64)


def fit_linear(X, y):
    """Ridge-stabilised least squares (reading R20): standardise the columns on the data, drop
    constant ones, solve (Z^T Z + 1e-6 I) g = Z^T (y - ybar); -> (beta0, beta[p])."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n, p = X.shape
    ybar = float(np.sum(y)) / n
    beta = np.zeros(p)
    if p:
        mu = np.sum(X, axis=0) / n
        sd = np.sqrt(np.sum((X - mu) ** 2, axis=0) / n)
        keep = sd > 1e-9 * np.maximum(1.0, np.abs(mu))
        if keep.any():
            Z = (X[:, keep] - mu[keep]) / sd[keep]
            A = Z.T @ Z + RIDGE * np.eye(int(keep.sum()))
            g = np.linalg.solve(A, Z.T @ (y - ybar))
            beta[keep] = g / sd[keep]
        beta0 = ybar - float(beta @ mu)
    else:
        beta0 = ybar
    return beta0, beta


def r_squared(y, yhat):
    """1 - SS_res / SS_tot; zero variance -> 0 (S:403 convention)."""
    y = np.asarray(y, dtype=np.float64)
    sst = float(np.sum((y - np.sum(y) / len(y)) ** 2))
    if sst <= 1e-24 * float(np.sum(y * y)):
        return 0.0
    return 1.0 - float(np.sum((y - yhat) ** 2)) / sst


def weights(r2):
    """Appendix B: w_i = max(0, R^2_i) / sum_j max(0, R^2_j); None = Unavailable."""
    pos = [max(0.0, float(r)) for r in r2]
    tot = sum(pos)
    if tot <= 0.0:
        return None
    return [p / tot for p in pos]


def holdout_split(n, seed):
    keys = [splitmix64(seed ^ 0xE45E ^ i) for i in range(n)]
    order = sorted(range(n), key=lambda i: keys[i])
    nh = max(1, n // 5)
    hold = sorted(order[:nh])
    train = sorted(order[nh:])
    return train, hold


class Ensemble:
    """Fitted ensemble: per model (name, cols, beta0, beta, R^2); weights or None (Unavailable)."""

    def __init__(self, space, digits, cost, seed=0):
        y = np.log(np.asarray(cost, dtype=np.float64))
        n = len(y)
        train, hold = holdout_split(n, seed)
        self.models = []
        r2 = []
        for name, knobs in TABLE2:
            cols = subset_features(space, knobs)
            if len(train) < len(cols) + 2 or not hold:
                self.models.append((name, cols, 0.0, np.zeros(len(cols)), -np.inf))
                r2.append(-np.inf)
                continue
            Xt = encode(space, [digits[i] for i in train], cols)
            b0, b = fit_linear(Xt, y[train])
            Xh = encode(space, [digits[i] for i in hold], cols)
            r = r_squared(y[hold], b0 + Xh @ b)
            self.models.append((name, cols, b0, b, r))
            r2.append(r)
        self.r2 = r2
        self.w = weights(r2)

    @property
    def available(self):
        return self.w is not None

    def predict(self, space, digits):
        """ln-cost prediction sum_i w_i yhat_i(x) (the Appendix B ensemble in ln units)."""
        out = np.zeros(len(digits))
        for (name, cols, b0, b, r), w in zip(self.models, self.w):
            if w == 0.0:
                continue
            out += w * (b0 + encode(space, digits, cols) @ b)
        return out
