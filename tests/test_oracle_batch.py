"""Pins for oracle/batch.py and oracle/parallel.py, plus the oracle pins the round-1 review found
missing (not gpu).

  * batch forms == scalar forms of the oracle, element by element (Feistel, CVI unrank, knob
    arrays + simulator, features, cross-covariance, posterior);
  * SURVEY Appendix C counts N_valid for C5 (5,000,756) and C4 (153,494,963; slow, AS_SLOW=1),
    produced by an independent nested-loop enumerator during the survey, not by oracle/;
  * gp.features by hand on configurations with gated-off features (reading R9: phi =
    digit_eff / (n - 1), inactive -> default digit; x~ = phi / l);
  * the fit's prior offset b = mean(y - m0) and incumbent f* = min y on a 3-point set whose
    residuals are chosen (reading R9).
"""

import math
import os

import numpy as np
import pytest

from conftest import cfg_digits, golden, space_path
from oracle import batch as B, feistel as F, gp, parallel as PAR, run, sim, space as S

PRESETS = ("P0", "C1", "C2", "C3", "C4", "C5")


@pytest.fixture(scope="module")
def spaces():
    return {n: S.load_space(space_path(n)) for n in PRESETS}


@pytest.mark.parametrize("n", [1, 2, 3, 5, 1000, (1 << 20) - 3, 356925584, 5550148])
@pytest.mark.parametrize("seed", [0, 7])
def test_feistel_batch_equals_scalar(n, seed):
    f = F.Feistel(n, seed)
    j = np.unique(np.linspace(0, n - 1, num=min(n, 2000)).astype(np.int64))
    got = B.feistel_batch(n, seed, j)
    assert [f(int(x)) for x in j] == got.tolist()


@pytest.mark.parametrize("name", ["P0", "C1", "C3"])
def test_unrank_batch_full_enumeration(spaces, name):
    # every CVI position of the space, against the scalar DP's enumeration order
    o = spaces[name]
    dg, act, raw = B.Unranker(o).unrank(np.arange(o.n_cvi()))
    ref = list(o.enumerate_cvi())
    assert dg.tolist() == ref
    assert raw.tolist() == [o.encode_raw(d) for d in ref]
    assert act.tolist() == [o.activity(d) for d in ref]


@pytest.mark.parametrize("name", ["C2", "C4", "C5"])
def test_unrank_batch_samples(spaces, name):
    o = spaces[name]
    rng = np.random.default_rng(3)
    p = np.concatenate([[0, o.n_cvi() - 1], rng.integers(0, o.n_cvi(), 400)])
    dg, act, raw = B.Unranker(o).unrank(p)
    for i, q in enumerate(p):
        d = o.cvi_unrank(int(q))
        assert dg[i].tolist() == d and raw[i] == o.encode_raw(d) and act[i].tolist() == o.activity(d)


@pytest.mark.parametrize("name", PRESETS)
def test_sim_features_batch_bitwise(spaces, name):
    o = spaces[name]
    rng = np.random.default_rng(5)
    p = rng.integers(0, o.n_cvi(), 300)
    dg, act, raw = B.Unranker(o).unrank(p)
    dl = [list(map(int, d)) for d in dg]
    c1, ok1, m1 = sim.simulate(o, dl)
    c2, ok2, m2 = B.simulate(o, dg, act)
    assert np.array_equal(ok1, ok2) and np.array_equal(m1, m2) and np.array_equal(c1, c2)
    assert np.array_equal(gp.features(o, dl), B.features(o, dg, act))


@pytest.mark.parametrize("kernel", ["matern52", "rbf"])
def test_posterior_batch_equals_scalar(spaces, kernel):
    o = S.load_space(dict(spaces["C2"].doc, gp=dict(spaces["C2"].gp, kernel=kernel)))
    rng = np.random.default_rng(11)
    U = B.Unranker(o)
    pos = rng.integers(0, o.n_cvi(), 200)
    dg, act, raw = U.unrank(pos)
    ok = B.simulate(o, dg, act)[1]
    obs = [list(map(int, d)) for d, v in zip(dg[:80], ok[:80]) if v][:24]
    cs = sim.simulate(o, obs)[0] * np.exp(0.1 * rng.normal(size=len(obs)))
    fit = run.observed_fit(o, [o.encode_raw(d) for d in obs], cs)
    X = B.features(o, dg[100:], act[100:])
    m0 = rng.normal(size=len(X))
    mu1, s21, _ = fit.posterior(X, m0)
    mu2, s22 = B.posterior(fit, X, m0)
    assert np.allclose(mu1, mu2, rtol=0, atol=1e-13) and np.allclose(s21, s22, rtol=0, atol=1e-13)


def test_parallel_topk_equals_scalar_run(spaces):
    # the sharded batch oracle reproduces oracle/run.py's exact top-k (C2, whole space in RANGE)
    o = spaces["C2"]
    rng = np.random.default_rng(2)
    U = B.Unranker(o)
    dg, act, raw = U.unrank(rng.integers(0, o.n_cvi(), 400))
    ok = B.simulate(o, dg, act)[1]
    obs = [list(map(int, d)) for d, v in zip(dg, ok) if v][:16]
    fit = run.observed_fit(o, [o.encode_raw(d) for d in obs], sim.simulate(o, obs)[0] * 1.1)
    ref = run.topk(run.score_batch(o, fit, "range", 0, o.n_cvi(), acq="ei"), 40)
    got, nval = PAR.topk(o, fit, "range", 0, o.n_cvi(), 40, acq="ei", procs=4)
    assert [r for r, _ in got] == [r for r, _ in ref]
    assert np.allclose([s for _, s in got], [s for _, s in ref], rtol=0, atol=1e-12)
    assert nval == golden("counts.json")["C2"]["n_valid"]


def test_n_valid_C5(spaces):
    assert PAR.count_valid(spaces["C5"]) == golden("counts.json")["C5"]["n_valid"]


@pytest.mark.skipif(not os.environ.get("AS_SLOW"), reason="3.6e8 positions (~5 min on 8 cores); AS_SLOW=1")
def test_n_valid_C4(spaces):
    assert PAR.count_valid(spaces["C4"]) == golden("counts.json")["C4"]["n_valid"]


# ---------------------------------------------------------------- hand-computed pins
def test_features_by_hand_P0_gated_off(spaces):
    # P0, l = 0.5 so x~ = 2 phi.  tp = 1 gates off sp and tp_comm; their raw digits
    # are deliberately NOT the default here (1 and 5): the feature map must use the default digit
    o = spaces["P0"]
    dg = cfg_digits(o, {"pp": 2, "tp": 1, "dp": 4, "ep": 1, "cp": 1, "ar": True, "mbs": 4, "ddp": 2,
                        "ddp_bucket": 5})
    dg[o.index["sp"]] = 1
    dg[o.index["tp_comm"]] = 5
    # pp 1/3, tp 0, dp 2/3, ep 0, cp 0, sp (default) 0, ar 1/1, mbs 2/3, ddp 1/3, tp_comm 0, bucket 4/7
    want = 2.0 * np.array([1 / 3, 0, 2 / 3, 0, 0, 0, 1, 2 / 3, 1 / 3, 0, 4 / 7])
    assert np.allclose(gp.features(o, [dg])[0], want, rtol=0, atol=1e-15)


def test_features_by_hand_C4_gated_off(spaces):
    # C4: ar = none gates off arl (raw digit 3 here, not the default 0); vpp active (pp > 1),
    # sp/tpov/tp_comm active (tp > 1, sp, tpov), dopt/ovp/ovg/bucket/ddp active (dp > 1, dopt)
    o = spaces["C4"]
    dg = cfg_digits(o, {"pp": 4, "vpp": 2, "tp": 8, "dp": 8, "cp": 1, "mbs": 2, "ar": "none", "sp": True,
                        "tpov": True, "tp_comm": 10, "dopt": True, "ovp": False, "ovg": True, "ddp_bucket": 33,
                        "ddp": 16})
    dg[o.index["arl"]] = 3
    phi = [2 / 6, 1 / 3, 3 / 3, 3 / 8, 0, 1 / 3, 0, 0, 1, 1, 6 / 32, 1, 0, 1, 32 / 63, 4 / 8]
    assert np.allclose(gp.features(o, [dg])[0], 2.0 * np.array(phi), rtol=0, atol=1e-15)


def test_fit_offset_and_incumbent_by_hand(spaces):
    # three valid C1 configurations profiled at cost_sim * e^delta, delta = (0.1, -0.2, 0.4):
    # y - m0 = delta, so b = mean(delta) = 0.1, residuals (0, -0.3, 0.3), f* = min ln c
    o = spaces["C1"]
    dl = [o.cvi_unrank(p) for p in (3, 50, 120)]
    raws = [o.encode_raw(d) for d in dl]
    cs_sim = sim.simulate(o, dl)[0]
    delta = np.array([0.1, -0.2, 0.4])
    costs = cs_sim * np.exp(delta)
    fit = run.observed_fit(o, raws, costs)
    assert fit.b == pytest.approx(0.1, abs=1e-14)
    assert np.allclose(fit.res, [0.0, -0.3, 0.3], rtol=0, atol=1e-14)
    assert fit.fstar == min(math.log(c) for c in costs)
