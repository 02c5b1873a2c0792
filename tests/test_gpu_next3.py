"""NEXT-3 on the GPU (-m gpu): Algorithm 1's top-K re-evaluation at the fidelity switch
drawn from the certified top-K of the WHOLE space under the simulator -- the scoring hot path
(score_batch SIM + topk) -- equals the oracle's exact top-K over every configuration, and the run
ends at least as good as the best re-evaluated configuration."""

import math

import numpy as np
import pytest

from conftest import space_path
from oracle import parallel as OP, run as orun
from parity_util import oracle_space

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
A = pytest.importorskip("paper_2603_11603_b200.autoscout")
from paper_2603_11603_b200 import search as SE  # noqa: E402
from test_next3_search import truth  # noqa: E402


@pytest.mark.parametrize("name", ["C2", "P0"])
def test_switch_reevaluates_certified_gpu_topk(name):
    sp = A.Space(space_path(name), 0)
    real = truth(sp)
    cfg = SE.RunConfig(T=20, tau=5, seed=3, K_reval=5, gpu_topk=True)
    r = SE.run(sp, real, cfg, sim_cost=lambda x: 3.0 * real(x))      # forces the switch at t = 5
    sw = [e for e in r["trace"] if e.get("event") == "switch"]
    assert len(sw) == 1
    o = oracle_space(name)
    fit = orun.observed_fit(o, [], [])
    ref, _ = OP.topk(o, fit, "range", 0, o.n_cvi(), 5, acq="sim")
    assert sw[0]["reval"] == [raw for raw, _ in ref]
    assert r["best_cost"] <= min(real(x) for x in sw[0]["reval"]) + 1e-12
    assert math.isfinite(r["best_cost"])
