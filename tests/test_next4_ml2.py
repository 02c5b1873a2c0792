"""NEXT-4: GP hyper-parameter evidence (ML-II), on the CPU (not gpu): the oracle's
log marginal likelihood pinned against a closed form (M = 1) and a library multivariate-normal
density (scipy), the search-point sampler against its definition; the C-ABI entry points exist
and reject bad input.  The device kernel is checked against the oracle in test_gpu_next4.py."""

import math

import numpy as np
import pytest

from oracle import gp
from parity_util import observed
from oracle import run

A = pytest.importorskip("paper_2603_11603_b200.autoscout")


def test_lml_single_observation_closed_form(oracle_spaces):
    o = oracle_spaces["C1"]
    P = np.zeros((1, len(o.features)))
    for res, sf2, sn2 in [(0.3, 0.1, 1e-3), (-1.2, 2.0, 0.5)]:
        v = sf2 + sn2
        want = -0.5 * res * res / v - 0.5 * math.log(2 * math.pi * v)
        got = gp.log_marginal_likelihood(o, P, np.array([res]), np.ones(len(o.features)), sf2, sn2)
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want))


def test_lml_matches_scipy_mvn(oracle_spaces):
    stats = pytest.importorskip("scipy.stats")
    o = oracle_spaces["C2"]
    raws, costs = observed(o, 12, 0)
    fit = run.observed_fit(o, raws, costs)
    dg = [o.decode_raw(int(r)) for r in raws]
    P = gp.phi_matrix(o, dg)
    rng = np.random.default_rng(0)
    for _ in range(5):
        ls = np.exp(rng.uniform(np.log(0.2), np.log(3), len(o.features)))
        sf2, sn2 = float(np.exp(rng.uniform(-3, 1))), float(np.exp(rng.uniform(-8, -2)))
        X = P / ls
        r = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
        K = sf2 * (1 + math.sqrt(5) * r + 5 / 3 * r * r) * np.exp(-math.sqrt(5) * r) + sn2 * np.eye(len(dg))
        want = stats.multivariate_normal(mean=np.zeros(len(dg)), cov=K).logpdf(fit.res)
        got = gp.log_marginal_likelihood(o, P, fit.res, ls, sf2, sn2)
        assert abs(got - want) <= 1e-9 * max(1.0, abs(want))


def test_ml2_candidates_in_range(oracle_spaces):
    o = oracle_spaces["C4"]
    d = len(o.features)
    c0 = gp.ml2_candidate(o, 7, 0, np.full(d, 0.5), 0.1, 1e-3)
    assert np.allclose(c0, np.concatenate([np.full(d, 0.5), [0.1, 1e-3]]))
    for h in range(1, 200):
        c = gp.ml2_candidate(o, 7, h, None, None, None)
        assert np.all((c[:d] >= 0.1) & (c[:d] <= 10)) and 1e-3 <= c[d] <= 10
        assert 1e-6 * c[d] <= c[d + 1] <= 1e-1 * c[d]


def test_c_abi_rejects_bad_input():
    from conftest import space_path
    sp = A.Space(space_path("C1"), -1)
    with pytest.raises(A.AutoscoutError):
        sp.gp_lml(np.ones((2, sp.d + 2)))              # host-only handle cannot launch
    with pytest.raises(A.AutoscoutError):
        sp.set_gp_hyper(np.zeros(sp.d), 0.1, 1e-3)     # non-positive lengthscale
    sp.set_gp_hyper(np.full(sp.d, 0.7), 0.2, 1e-3)     # accepted, refits (no observations yet)
