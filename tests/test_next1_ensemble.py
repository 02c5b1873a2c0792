"""NEXT-1: the paper's regression-simulator ensemble as the GP prior mean, on the CPU.

Oracle pins (oracle/ensemble.py) against what PAPER.md / SPEC.md and the mathematics fix:
  * the Appendix B weight equation on SPEC's worked example (S:617 acceptance 1), the single-model
    and all-non-positive cases;
  * least squares: exact recovery of a linear law ("R^2 = 1.0"), the hand-solved 3-point
    example (S:404 slope 2, intercept 0), zero-variance R^2 = 0, agreement with
    numpy.linalg.lstsq (a library OLS) on well-posed data -- the 1e-6 ridge of reading R20 is
    within 1e-5 of OLS there;
  * Table 2 subsets mapped onto the presets' knob names.
Then the library's host fit (autoscout_ensemble_info / autoscout_prior / observe_info) against the
oracle on every preset, with the synthetic observed set and with a linear ln-cost law where all
four simulators are available.
"""

import json
import math

import numpy as np
import pytest

from conftest import space_text
from oracle import ensemble as E, run, sim
from parity_util import observed

A = pytest.importorskip("paper_2603_11603_b200.autoscout")

PRESETS = ("P0", "C1", "C2", "C3", "C4", "C5")


# ------------------------------------------------------------------ oracle pins
def test_weights_spec_example():
    w = E.weights([0.8, 0.2, -0.1, 0.1])
    for a, b in zip(w, [8 / 11, 2 / 11, 0.0, 1 / 11]):
        assert abs(a - b) <= 1e-12
    assert E.weights([0.5]) == [1.0]
    assert E.weights([0.0, -0.3, -1.0, -np.inf]) is None


def test_fit_linear_recovers_a_linear_law():
    rng = np.random.default_rng(0)
    X = rng.uniform(-2, 5, size=(40, 5))
    beta = np.array([0.3, -1.2, 0.05, 2.0, -0.7])
    y = 1.7 + X @ beta
    b0, b = E.fit_linear(X, y)
    assert abs(b0 - 1.7) < 1e-5 and np.allclose(b, beta, rtol=1e-5, atol=1e-6)
    Xh = rng.uniform(-2, 5, size=(10, 5))
    assert abs(E.r_squared(1.7 + Xh @ beta, b0 + Xh @ b) - 1.0) < 1e-9


def test_fit_linear_three_point_example():
    b0, b = E.fit_linear(np.array([[1.0], [2.0], [3.0]]), np.array([2.0, 4.0, 6.0]))
    assert abs(b[0] - 2.0) < 1e-6 and abs(b0) < 1e-5


def test_r_squared_zero_variance_is_zero():
    assert E.r_squared(np.array([3.0, 3.0, 3.0]), np.array([1.0, 2.0, 3.0])) == 0.0


def test_fit_linear_matches_lstsq():
    rng = np.random.default_rng(4)
    X = rng.normal(size=(60, 7)) * np.array([1, 10, 100, 0.1, 3, 7, 1])
    y = rng.normal(size=60)
    b0, b = E.fit_linear(X, y)
    D = np.hstack([np.ones((60, 1)), X])
    ref, *_ = np.linalg.lstsq(D, y, rcond=None)
    assert abs(b0 - ref[0]) <= 1e-5 * max(1, abs(ref[0]))
    assert np.allclose(b, ref[1:], rtol=1e-5, atol=1e-7)


def test_constant_columns_dropped():
    X = np.array([[1.0, 4.0], [2.0, 4.0], [3.0, 4.0], [5.0, 4.0]])
    b0, b = E.fit_linear(X, 2 * X[:, 0] + 1)
    assert b[1] == 0.0 and abs(b[0] - 2) < 1e-6


def test_table2_subsets_on_presets(oracle_spaces):
    c4 = oracle_spaces["C4"]
    names = lambda cols: [c4.features[j].name for j in cols]
    assert names(E.subset_features(c4, E.TABLE2[0][1])) == ["pp", "tp", "dp", "mbs"]
    assert "dopt" in names(E.subset_features(c4, E.TABLE2[2][1]))
    assert set(names(E.subset_features(c4, E.TABLE2[3][1]))) == {"pp", "tp", "dp", "mbs", "ar", "tp_comm"}
    p0 = oracle_spaces["P0"]
    assert "ddp" in [p0.features[j].name for j in E.subset_features(p0, E.TABLE2[2][1])]


def test_holdout_split():
    for n in (1, 4, 5, 16, 33, 256):
        tr, ho = E.holdout_split(n, 0)
        assert len(ho) == max(1, n // 5) and sorted(tr + ho) == list(range(n))


# ------------------------------------------------------------------ library vs oracle (host)
def ens_doc(name, seed=0):
    doc = json.loads(space_text(name))
    doc.setdefault("gp", {})
    doc["gp"]["prior"] = "ensemble"
    doc["gp"]["ensemble_seed"] = seed
    return doc


def linear_law_costs(o, raws):
    """ln c = 0.4 + small multiples of the knobs every Table 2 simulator shares (mbs, tp, pp, dp;
    test input, not the method): each simulator explains it, so all four are available."""
    out = []
    for r in raws:
        dg = o.decode_raw(int(r))
        s = 0.4
        for j, f in enumerate(o.features):
            if f.name in ("tp", "pp", "dp", "mbs"):
                s += 0.01 * (j + 1) * f.numeric(dg[j])
        out.append(math.exp(s))
    return out


def _compare(name, doc, raws, costs):
    from oracle import space as S
    o = S.load_space(doc)
    sp = A.Space(doc, -1)
    sp.observe(raws, costs)
    fit = run.observed_fit(o, raws, costs)
    digits = [o.decode_raw(int(r)) for r in raws]
    ens = E.Ensemble(o, digits, costs, doc["gp"]["ensemble_seed"])
    r2, w, av = sp.ensemble_info()
    assert av == ens.available
    for a, b in zip(r2, ens.r2):
        assert (a == b == -np.inf) or abs(a - b) <= 1e-8 * max(1.0, abs(b))
    if av:
        for a, b in zip(w, ens.w):
            assert abs(a - b) <= 1e-8
    m, bb, fstar = sp.observe_info()
    assert abs(bb - fit.b) <= 1e-9 * max(1.0, abs(fit.b))
    rng = np.random.default_rng(1)
    n = o.n_cvi()
    ps = rng.integers(0, n, 200)
    dgs = [o.cvi_unrank(int(p)) for p in ps]
    want = ens.predict(o, dgs) if av else np.log(sim.simulate(o, dgs)[0])
    for dg, m0 in zip(dgs, want):
        got, src = sp.prior(o.encode_raw(dg))
        assert src == (1 if av else 0)
        assert abs(got - m0) <= 1e-9 * max(1.0, abs(m0))
    return av


@pytest.mark.parametrize("name,M", [("P0", 16), ("C1", 16), ("C2", 64), ("C3", 32), ("C4", 256), ("C5", 128)])
def test_library_ensemble_matches_oracle_synthetic(oracle_spaces, name, M):
    raws, costs = observed(oracle_spaces[name], M, 0)
    _compare(name, ens_doc(name), raws, costs)


@pytest.mark.parametrize("name,M", [("C1", 16), ("C2", 64), ("C4", 256), ("C5", 128), ("P0", 16)])
def test_library_ensemble_matches_oracle_linear_law(oracle_spaces, name, M):
    o = oracle_spaces[name]
    raws, _ = observed(o, M, 0)
    costs = linear_law_costs(o, raws)
    assert _compare(name, ens_doc(name, seed=3), raws, costs)     # every preset: ensemble available


def test_prior_sim_by_default(oracle_spaces):
    o = oracle_spaces["C2"]
    sp = A.Space(json.loads(space_text("C2")), -1)
    raws, costs = observed(o, 64, 0)
    sp.observe(raws, costs)
    assert sp.ensemble_info()[2] is False
    dg = o.cvi_unrank(77)
    m0, src = sp.prior(o.encode_raw(dg))
    assert src == 0 and abs(m0 - float(np.log(sim.simulate(o, [dg])[0][0]))) <= 1e-12


def test_bad_prior_rejected():
    doc = json.loads(space_text("C1"))
    doc.setdefault("gp", {})["prior"] = "mlr"
    with pytest.raises(A.AutoscoutError):
        A.Space(doc, -1)
