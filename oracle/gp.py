"""Oracle: GP surrogate on the log-cost residual over the simulator prior.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper has no GP (it argues against global surrogates); north_star
mandates "the surrogate posterior mean/variance ... against the already-profiled set", in
the lineage of the BO baseline CherryPick.  Reading R9 (SURVEY
ledger #1 and Appendix A.5):

  phi_j  = digit_eff_j / (n_j - 1)  (0 if n_j == 1);   x~_j = phi_j / l_j
  k(x,o) = sf2 (1 + sqrt5 r + 5/3 r^2) exp(-sqrt5 r),  r = ||x~ - o~||_2   [RBF: sf2 exp(-r^2/2)]
  observe: y_i = ln c_i,  m0 = ln cost_sim,  b = mean(y - m0(o)),  res = y - m0(o) - b,
           K = [k(o_i,o_j)] + sn2 I,  alpha = K^-1 res,  f* = min_i y_i
  mu     = m0(x) + b + k*^T alpha
  s2     = max(sf2 - k*^T K^-1 k*, 0)

Computed by a dense direct solve (numpy.linalg.solve) -- the plain definition; the CUDA
library uses Cholesky + L^-1 instead.
"""

from __future__ import annotations

import math

import numpy as np

SQRT5 = math.sqrt(5.0)


def lengthscales(space):
    ls = space.gp.get("lengthscale", 1.0)
    d = len(space.features)
    if isinstance(ls, (int, float)):
        return np.full(d, float(ls))
    ls = np.asarray(ls, dtype=np.float64)
    assert ls.shape == (d,)
    return ls


def features(space, digits_list):
    """x~ for a batch of configurations (inactive features encoded at their default)."""
    ls = lengthscales(space)
    X = np.zeros((len(digits_list), len(space.features)), dtype=np.float64)
    for b, dg in enumerate(digits_list):
        act = space.activity(dg)
        for j, f in enumerate(space.features):
            de = dg[j] if act[j] else f.default_digit
            phi = de / (f.n - 1) if f.n > 1 else 0.0
            X[b, j] = phi / ls[j]
    return X


def kernel_r(space, r):
    sf2 = float(space.gp["sf2"])
    kind = space.gp.get("kernel", "matern52")
    if kind == "matern52":
        return sf2 * (1.0 + SQRT5 * r + (5.0 / 3.0) * r * r) * np.exp(-SQRT5 * r)
    if kind == "rbf":
        return sf2 * np.exp(-0.5 * r * r)
    raise ValueError(kind)


def cross_cov(space, X, O):
    """k(x_b, o_i) by direct differences (no ||x||^2+||o||^2-2x.o expansion)."""
    diff = X[:, None, :] - O[None, :, :]
    r = np.sqrt(np.sum(diff * diff, axis=2))
    return kernel_r(space, r)


class Fit:
    """The fitted GP of one observed set (SURVEY §8(a) a-obs)."""

    def __init__(self, space, O, y, m0_obs):
        self.space = space
        self.O = np.asarray(O, dtype=np.float64)
        self.M = self.O.shape[0]
        self.sf2 = float(space.gp["sf2"])
        self.sn2 = float(space.gp["sn2"])
        self.y = np.asarray(y, dtype=np.float64)
        self.m0_obs = np.asarray(m0_obs, dtype=np.float64)
        if self.M == 0:
            self.b = 0.0
            self.fstar = math.inf
            self.K = np.zeros((0, 0))
            self.alpha = np.zeros(0)
            return
        resid0 = self.y - self.m0_obs
        self.b = float(np.mean(resid0))
        self.res = resid0 - self.b
        self.K = cross_cov(space, self.O, self.O) + self.sn2 * np.eye(self.M)
        self.alpha = np.linalg.solve(self.K, self.res)
        self.fstar = float(np.min(self.y))

    def posterior(self, X, m0):
        """-> (mu, s2, kstar) for candidates with features X [B,d] and prior means m0 [B]."""
        X = np.asarray(X, dtype=np.float64)
        m0 = np.asarray(m0, dtype=np.float64)
        if self.M == 0:
            return m0 + 0.0, np.full(len(m0), self.sf2), np.zeros((len(m0), 0))
        mu = np.empty(len(m0))
        s2 = np.empty(len(m0))
        ks_all = []
        for lo in range(0, len(m0), 2048):                    # chunks bound memory only
            ks = cross_cov(self.space, X[lo:lo + 2048], self.O)          # [B, M]
            mu[lo:lo + 2048] = m0[lo:lo + 2048] + self.b + ks @ self.alpha
            sol = np.linalg.solve(self.K, ks.T)                          # K^-1 k*, [M, B]
            quad = np.sum(ks.T * sol, axis=0)
            s2[lo:lo + 2048] = np.maximum(self.sf2 - quad, 0.0)
            if len(m0) <= 4096:
                ks_all.append(ks)
        ks = np.concatenate(ks_all) if ks_all else None
        return mu, s2, ks


def fit_observed(space, digits_list, cost_obs, cost_sim_obs):
    """observe(): y = ln c, m0 = ln cost_sim."""
    O = features(space, digits_list) if len(digits_list) else np.zeros((0, len(space.features)))
    return Fit(space, O, np.log(np.asarray(cost_obs, dtype=np.float64)),
               np.log(np.asarray(cost_sim_obs, dtype=np.float64)))


def fit_observed_prior(space, digits_list, cost_obs, m0_obs):
    """observe() with an explicit prior mean at the observed points (NEXT-1 ensemble, R20)."""
    O = features(space, digits_list) if len(digits_list) else np.zeros((0, len(space.features)))
    return Fit(space, O, np.log(np.asarray(cost_obs, dtype=np.float64)), np.asarray(m0_obs, dtype=np.float64))


# ---------------------------------------------------------------- NEXT-4: ML-II evidence (reading R21)
def phi_matrix(space, digits_list):
    """phi_j = effective digit / (n_j - 1) of each observed configuration (lengthscale-free)."""
    P = np.zeros((len(digits_list), len(space.features)), dtype=np.float64)
    for b, dg in enumerate(digits_list):
        act = space.activity(dg)
        for j, f in enumerate(space.features):
            de = dg[j] if act[j] else f.default_digit
            P[b, j] = de / (f.n - 1) if f.n > 1 else 0.0
    return P


def log_marginal_likelihood(space, P, res, ls, sf2, sn2):
    """ln N(res; 0, K) with K_ij = k(||(phi_i - phi_j) / l||) + sn2 delta_ij (the definition:
    -1/2 res^T K^-1 res - 1/2 ln det K - M/2 ln 2 pi, by numpy slogdet and solve)."""
    X = P / np.asarray(ls, dtype=np.float64)[None, :]
    diff = X[:, None, :] - X[None, :, :]
    r = np.sqrt(np.sum(diff * diff, axis=2))
    kind = space.gp.get("kernel", "matern52")
    if kind == "matern52":
        K = sf2 * (1.0 + SQRT5 * r + (5.0 / 3.0) * r * r) * np.exp(-SQRT5 * r)
    else:
        K = sf2 * np.exp(-0.5 * r * r)
    K = K + sn2 * np.eye(len(res))
    sign, logdet = np.linalg.slogdet(K)
    if sign <= 0:
        return -math.inf
    return float(-0.5 * res @ np.linalg.solve(K, res) - 0.5 * logdet - 0.5 * len(res) * math.log(2 * math.pi))


def ml2_candidate(space, seed, h, ls0, sf20, sn20):
    """ML-II search point h (R21): h = 0 the current setting; else log-uniform draws from the
    counter-based uniforms u_k = (splitmix64(seed ^ 0x3111 ^ (64 h + k)) >> 11) * 2^-53."""
    from .feistel import splitmix64
    d = len(space.features)
    if h == 0:
        return np.concatenate([np.asarray(ls0, dtype=np.float64), [sf20, sn20]])
    u = [(splitmix64(seed ^ 0x3111 ^ (64 * h + k)) >> 11) * 2.0 ** -53 for k in range(d + 2)]
    ls = [math.exp(math.log(0.1) + u[j] * math.log(100.0)) for j in range(d)]
    sf2 = math.exp(math.log(1e-3) + u[d] * math.log(1e4))
    sn2 = sf2 * math.exp(math.log(1e-6) + u[d + 1] * math.log(1e5))
    return np.array(ls + [sf2, sn2])
