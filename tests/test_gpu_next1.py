"""GPU parity with the regression-simulator ensemble as the GP prior mean (NEXT-1, -m gpu):
every kernel path that forms m0 (generation kernel, SIMT and tensor-core score kernels, FP64
refine) against the oracle, element by element (bars: DESIGN.md §4.3)."""

import json

import numpy as np
import pytest

from conftest import space_text
from oracle import run, space as S
from parity_util import ei_tolerance_ok, observed
from test_next1_ensemble import linear_law_costs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
A = pytest.importorskip("paper_2603_11603_b200.autoscout")


def _doc(name):
    doc = json.loads(space_text(name))
    doc.setdefault("gp", {})["prior"] = "ensemble"
    doc["gp"]["ensemble_seed"] = 3
    return doc


def _run(sp, mode, begin, n, seed, acq, kappa=None, k=32):
    sc = torch.empty(n, dtype=torch.float32, device="cuda")
    rw = torch.empty(n, dtype=torch.int64, device="cuda")
    sp.score_batch(mode=mode, begin=begin, count=n, seed=seed, acq=acq, kappa=kappa, k=k, d_scores=sc, d_raw=rw)
    top = sp.topk(k)
    torch.cuda.synchronize()
    return sc.cpu().numpy(), rw.cpu().numpy().astype(np.uint64), top


CASES = [("C3", 32, "range", None, "linear"), ("C2", 64, "range", None, "linear"),
         ("C5", 128, "sample", 40000, "linear"), ("C4", 256, "sample", 40000, "synthetic")]


@pytest.mark.parametrize("name,M,mode,count,law", CASES)
@pytest.mark.parametrize("path", ["auto", "simt"])
def test_ensemble_prior_parity(name, M, mode, count, law, path):
    doc = _doc(name)
    o = S.load_space(doc)
    raws, costs = observed(o, M, 0)
    if law == "linear":
        costs = linear_law_costs(o, raws)
    fit = run.observed_fit(o, raws, costs)
    assert fit.ens is not None                      # the ensemble is the prior in every case
    n = o.n_cvi() if count is None else count
    rec = run.score_batch(o, fit, mode, 0, n, seed=0, acq="lcb", kappa=0.0)
    sp = A.Space(doc, 0)
    sp.observe(raws, costs)
    sp.set_path(path)
    assert sp.ensemble_info()[2]
    v = rec["valid"]
    # SIM = -m0: the prior itself
    sc, rw, top = _run(sp, mode, 0, n, 0, "sim")
    assert np.array_equal(rw, rec["raw"]) and np.array_equal(np.isfinite(sc), v)
    assert np.all(np.abs(-sc[v] - rec["m0"][v]) <= 1e-5 * np.maximum(1.0, np.abs(rec["m0"][v])))
    # posterior mean (LCB, kappa = 0)
    sc, rw, top = _run(sp, mode, 0, n, 0, "lcb", kappa=0.0)
    mu = rec["mu"]
    assert np.all(np.abs(-sc[v] - mu[v]) <= 1e-5 * np.maximum(1.0, np.abs(mu[v])))
    assert [r for r, _ in top] == [r for r, _ in run.topk(rec, 32)]
    # EI + certified top-k (FP64 refine uses the same prior)
    sc, rw, top = _run(sp, mode, 0, n, 0, "ei")
    ref = run.score_batch(o, fit, mode, 0, n, seed=0, acq="ei")
    ok = ei_tolerance_ok(sc[v].astype(np.float64), ref["score"][v], mu[v], rec["s2"][v], fit.fstar, fit.sf2)
    assert ok.all()
    want = run.topk(ref, 32)
    assert [r for r, _ in top] == [r for r, _ in want]
    for (_, a), (_, b) in zip(top, want):
        assert a == pytest.approx(b, rel=1e-12, abs=1e-12)
