"""Oracle: acquisition scores (higher is better).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Not in the paper (its UCB1 of Eq. 1, is the bandit's arm rule); north_star asks
for "the acquisition (EI/UCB)".  Reading R10 (ledger #11-13),
on the objective y = ln(cost), lower cost = better:

  EI (min form):  u = f* - mu - xi;  sigma = sqrt(s2)
                  sigma == 0 -> score = ln(max(u, 0))  (-inf if u <= 0)
                  else z = u / sigma, score = ln sigma + ln h(z),  h(z) = phi(z) + z Phi(z)
                  ln h(z) = ln(phi(z) + z Phi(z))                    for z >= -10
                          = -z^2/2 - ln(2 pi)/2 - 2 ln(-z)
                            + log1p(-3/z^2 + 15/z^4 - 105/z^6 + 945/z^8)   for z < -10
  LCB:            score = kappa * sigma - mu
  SIM:            score = -m0 = -ln cost_sim
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import erfc

LN_2PI = math.log(2.0 * math.pi)


def lnh(z):
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    hi = z >= -10.0
    zh = z[hi]
    phi = np.exp(-0.5 * zh * zh) / math.sqrt(2.0 * math.pi)
    Phi = 0.5 * erfc(-zh / math.sqrt(2.0))
    out[hi] = np.log(phi + zh * Phi)
    zl = z[~hi]
    z2 = zl * zl
    out[~hi] = (-0.5 * z2 - 0.5 * LN_2PI - 2.0 * np.log(-zl)
                + np.log1p(-3.0 / z2 + 15.0 / z2 ** 2 - 105.0 / z2 ** 3 + 945.0 / z2 ** 4))
    return out


def ei_score(mu, s2, fstar, xi=0.0):
    mu = np.asarray(mu, dtype=np.float64)
    s2 = np.asarray(s2, dtype=np.float64)
    u = fstar - mu - xi
    sigma = np.sqrt(s2)
    out = np.empty_like(mu)
    zero = sigma == 0.0
    with np.errstate(divide="ignore"):
        out[zero] = np.where(u[zero] > 0, np.log(np.where(u[zero] > 0, u[zero], 1.0)), -np.inf)
    nz = ~zero
    z = u[nz] / sigma[nz]
    out[nz] = np.log(sigma[nz]) + lnh(z)
    return out


def lcb_score(mu, s2, kappa):
    return kappa * np.sqrt(np.asarray(s2, dtype=np.float64)) - np.asarray(mu, dtype=np.float64)


def sim_score(m0):
    return -np.asarray(m0, dtype=np.float64)
