"""Pins for oracle/gp.py and oracle/acq.py (not gpu).

Pinned against things that are not the oracle's own routine:
  * Matern-5/2 and h(z) at high precision with mpmath (independent arithmetic);
  * the M=1 closed form of SURVEY §8(c);
  * the Schur-complement identity of the joint Gaussian (inverse of the (M+1)x(M+1) joint
    covariance) -- a different algorithm from the oracle's dense solve, which catches a
    dropped noise term, a wrong sign or a transposed operand;
  * noise-free interpolation (sigma_n^2 -> 0: posterior at an observed point -> its value);
  * EI by numerical integration of E[max(f* - xi - Y, 0)] (scipy.integrate.quad);
  * the sigma -> 0 limit and monotonicity of EI.
"""

import math

import mpmath as mp
import numpy as np
import pytest
from scipy.integrate import quad

from conftest import golden
from oracle import acq, gp

mp.mp.dps = 50
G = golden("gp_acq_values.json")


class _Sp:
    """Minimal stand-in space for the GP routines (features only need n and default)."""

    def __init__(self, sf2, sn2, kernel="matern52"):
        self.gp = {"sf2": sf2, "sn2": sn2, "kernel": kernel, "lengthscale": 1.0}
        self.features = []


def mp_matern(r, sf2=1.0):
    r = mp.mpf(r)
    return sf2 * (1 + mp.sqrt(5) * r + mp.mpf(5) / 3 * r * r) * mp.e ** (-mp.sqrt(5) * r)


def mp_h(z):
    z = mp.mpf(z)
    return mp.npdf(z) + z * mp.ncdf(z)


@pytest.mark.parametrize("r,val", [(float(k), v) for k, v in G["matern52_sf2_1"].items()])
def test_matern_values(r, val):
    got = gp.kernel_r(_Sp(1.0, 0.0), np.array([r]))[0]
    assert got == pytest.approx(float(mp_matern(r)), rel=1e-14)
    assert got == pytest.approx(val, abs=1e-10)


def test_gp_m1_closed_form():
    c = G["gp_M1"]
    sp = _Sp(c["sf2"], c["sn2"])
    fit = gp.Fit(sp, np.array([[0.0]]), np.array([c["residual"]]), np.array([0.0]))
    # b = mean(y - m0) absorbs a single residual; re-center so that res = 0.3 exactly
    fit.b = 0.0
    fit.res = np.array([c["residual"]])
    fit.alpha = np.linalg.solve(fit.K, fit.res)
    mu, s2, _ = fit.posterior(np.array([[c["r"]]]), np.array([0.0]))
    k = float(mp_matern(c["r"], mp.mpf(c["sf2"])))
    assert mu[0] == pytest.approx(k * c["residual"] / (c["sf2"] + c["sn2"]), rel=1e-13)
    assert mu[0] == pytest.approx(c["mu_minus_prior"], abs=1e-11)
    assert s2[0] == pytest.approx(c["s2"], abs=1e-11)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("kernel", ["matern52", "rbf"])
def test_gp_schur_complement(seed, kernel):
    rng = np.random.default_rng(seed)
    M, d = int(rng.integers(1, 9)), int(rng.integers(1, 5))
    sf2 = float(rng.uniform(0.01, 1.0))
    sn2 = sf2 * float(10 ** rng.uniform(-4, -1))
    sp = _Sp(sf2, sn2, kernel)
    O = rng.uniform(0, 2, size=(M, d))
    y = rng.normal(size=M)
    m0o = rng.normal(size=M)
    fit = gp.Fit(sp, O, y, m0o)
    X = rng.uniform(0, 2, size=(5, d))
    m0x = rng.normal(size=5)
    mu, s2, _ = fit.posterior(X, m0x)
    # joint covariance of (f(o_1..o_M) + noise, f(x)); conditional of the last coordinate
    for b in range(5):
        Z = np.vstack([O, X[b:b + 1]])
        diff = Z[:, None, :] - Z[None, :, :]
        r = np.sqrt((diff ** 2).sum(-1))
        Sig = gp.kernel_r(sp, r)
        Sig[:M, :M] += sn2 * np.eye(M)
        Pm = np.linalg.inv(Sig)
        s2_ref = 1.0 / Pm[M, M]
        mu_ref = m0x[b] + fit.b - (Pm[M, :M] @ (y - m0o - fit.b)) / Pm[M, M]
        assert s2[b] == pytest.approx(s2_ref, rel=1e-9, abs=1e-12 * sf2)
        assert mu[b] == pytest.approx(mu_ref, rel=1e-9, abs=1e-10)
        assert 0.0 <= s2[b] <= sf2


def test_gp_noise_free_interpolation():
    rng = np.random.default_rng(11)
    sp = _Sp(0.5, 1e-12)
    O = rng.uniform(0, 3, size=(6, 3))
    y = rng.normal(size=6)
    fit = gp.Fit(sp, O, y, np.zeros(6))
    mu, s2, _ = fit.posterior(O, np.zeros(6))
    assert np.allclose(mu, y, atol=1e-6)
    assert np.all(s2 < 1e-8)


@pytest.mark.parametrize("z", [0.0, 1.0, -1.0, -3.0, -6.0, -9.99, -10.0])
def test_lnh_direct_branch(z):
    assert acq.lnh(np.array([z]))[0] == pytest.approx(float(mp.log(mp_h(z))), rel=1e-12)


@pytest.mark.parametrize("z", [-10.01, -12.0, -20.0, -40.0])
def test_lnh_asymptotic_branch(z):
    # truncation error of the asymptotic series is below the next term 10395/z^10
    assert acq.lnh(np.array([z]))[0] == pytest.approx(float(mp.log(mp_h(z))), abs=1.2 * 10395 / z ** 10 + 1e-12)


def test_h_golden():
    for z, v in G["h"].items():
        assert float(mp_h(float(z))) == pytest.approx(v, rel=1e-9)
    assert acq.lnh(np.array([-10.0]))[0] == pytest.approx(G["ln_h_-10"], abs=1e-8)


@pytest.mark.parametrize("mu,s2,fstar,xi", [(0.1, 0.04, 0.2, 0.0), (0.5, 0.01, 0.2, 0.0), (-1.0, 0.3, 0.0, 0.05),
                                           (0.0, 1e-4, 0.03, 0.0), (2.0, 0.09, 1.0, 0.0)])
def test_ei_matches_integral(mu, s2, fstar, xi):
    sig = math.sqrt(s2)
    f = lambda y: max(fstar - xi - y, 0.0) * math.exp(-0.5 * ((y - mu) / sig) ** 2) / (sig * math.sqrt(2 * math.pi))
    ref, _ = quad(f, mu - 40 * sig, fstar - xi, epsabs=1e-300, epsrel=1e-12, limit=400)
    got = math.exp(acq.ei_score(np.array([mu]), np.array([s2]), fstar, xi)[0])
    assert got == pytest.approx(ref, rel=1e-8)


def test_ei_sigma_zero_limit():
    sc = acq.ei_score(np.array([0.1, 0.3]), np.array([0.0, 0.0]), 0.2)
    assert sc[0] == pytest.approx(math.log(0.1), rel=1e-13) and sc[1] == -np.inf
    small = acq.ei_score(np.array([0.1]), np.array([1e-20]), 0.2)[0]
    assert small == pytest.approx(math.log(0.1), rel=1e-9)


def test_ei_monotone():
    mus = np.linspace(-1, 1, 41)
    s = acq.ei_score(mus, np.full(41, 0.05), 0.0)
    assert np.all(np.diff(s) < 0)                                   # increasing in f* - mu
    s2 = np.linspace(1e-4, 1.0, 41)
    t = acq.ei_score(np.full(41, 0.2), s2, 0.0)
    assert np.all(np.diff(t) > 0)                                   # increasing in sigma


def test_lcb_sim():
    assert acq.lcb_score(np.array([1.0]), np.array([0.25]), 2.0)[0] == pytest.approx(0.0)
    assert acq.sim_score(np.array([math.log(2.0)]))[0] == pytest.approx(-math.log(2.0))
