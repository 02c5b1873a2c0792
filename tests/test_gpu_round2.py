"""GPU parity of the path the bench times, at full size, plus the round-1 review's open items (-m gpu).

  * full size, no per-candidate outputs (the bench configuration): C4's 10^8 SAMPLE batch and C5's
    whole space, certified top-32 set AND order == the oracle's exact top-32, computed over every
    candidate by the batch oracle on all host cores (oracle/parallel.py); valid counts exact;
  * the FP32 screen that admits candidates (d_screen: mu, sigma^2, screen, bound), compared row by
    row with the oracle: mu and sigma^2 at the SURVEY A.7 bars (|d mu| <= 1e-5 max(1, |mu|),
    |d s2| <= 1e-5 sf2), and the certified bound >= the oracle's exact score on every row
     -- C2 whole space, C4 and C5 windows;
  * k in {1, 7, 256, 1024} at M = 256 and 128 == oracle;
  * the sharded exchange (topk_pool on G handles with disjoint shares + topk_merge, SURVEY §4.2
    T3 "fake all-gather") == single-handle topk == oracle, G = 2 and 4;
  * kappa / xi validation, pool invalidation on refit, mixed-acquisition
    accumulate rejected, duplicate LIST positions, set_gp_hyper restore on failure.
"""

import math

import numpy as np
import pytest

from conftest import space_path
from oracle import batch as OB, feistel, parallel as OP, run
from parity_util import observed, oracle_space

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
A = pytest.importorskip("paper_2603_11603_b200.autoscout")

_C = {}


def setup(name, M, obs_seed=0):
    key = (name, M, obs_seed)
    if key not in _C:
        o = oracle_space(name)
        raws, costs = observed(o, M, obs_seed)
        fit = run.observed_fit(o, raws, costs)
        _C[key] = (o, fit, raws, costs)
    o, fit, raws, costs = _C[key]
    sp = A.Space(space_path(name), 0)
    if M:
        sp.observe(raws, costs)
    return o, fit, sp


def same_topk(got, ref):
    assert [r for r, _ in got] == [r for r, _ in ref]
    assert np.allclose([s for _, s in got], [s for _, s in ref], rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- full size, bench configuration
@pytest.mark.parametrize("name,M,mode,count", [("C4", 256, "sample", 100_000_000), ("C5", 128, "range", None)])
def test_full_size_topk_equals_oracle(name, M, mode, count):
    o, fit, sp = setup(name, M)
    count = o.n_cvi() if count is None else count
    vc = torch.zeros(1, dtype=torch.int64, device="cuda")
    sp.score_batch(mode=mode, begin=0, count=count, seed=0, acq="ei", k=32, d_valid_count=vc)
    top = sp.topk(32)                 # no d_scores: the FP32 screen + FP64 refine the bench runs
    torch.cuda.synchronize()
    ref, nval = OP.topk(o, fit, mode, 0, count, 32, seed=0, acq="ei")
    same_topk(top, ref)
    assert int(vc.item()) == nval


# ---------------------------------------------------------------- the FP32 screen, row by row
@pytest.mark.parametrize("name,M,mode,begin,count", [
    ("C2", 64, "range", 0, None),
    ("C4", 256, "sample", 3_000_000, 1 << 17),
    ("C5", 128, "range", 2_000_000, 1 << 17),
])
@pytest.mark.parametrize("acq", ["ei", "lcb"])
def test_fp32_screen_rows(name, M, mode, begin, count, acq):
    o, fit, sp = setup(name, M)
    sp.set_path("tc2")
    count = o.n_cvi() - begin if count is None else count
    scr = torch.full((count, 4), float("nan"), dtype=torch.float32, device="cuda")
    sp.score_batch(mode=mode, begin=begin, count=count, seed=0, acq=acq, k=32, d_screen=scr)
    sp.topk(32)
    torch.cuda.synchronize()
    g = scr.cpu().numpy().astype(np.float64)
    pos = (np.arange(begin, begin + count) if mode == "range"
           else OB.feistel_batch(o.n_cvi(), 0, np.arange(begin, begin + count)))
    rec = OP.score_positions(o, OB.Unranker(o), fit, pos, acq=acq, kappa=2.0)
    v = rec["valid"]
    assert np.array_equal(np.isfinite(g[:, 0]), v)
    mu, s2, screen, ub = g[v, 0], g[v, 1], g[v, 2], g[v, 3]
    # A.7: mu at 1e-5 max(1, |mu|), sigma^2 at 1e-5 sf2 -- read directly, not from LCB differences
    assert np.all(np.abs(mu - rec["mu"][v]) <= 1e-5 * np.maximum(1.0, np.abs(rec["mu"][v])))
    assert np.all(np.abs(s2 - rec["s2"][v]) <= 1e-5 * fit.sf2)
    # the admission key is an upper bound of the exact score on every row (certificate soundness)
    exact = rec["score"][v]
    fin = np.isfinite(exact)
    assert np.all(ub[fin] >= exact[fin])
    # and the FP32 screen itself is within its own margin of the exact score
    assert np.all(np.abs(screen[fin] - exact[fin]) <= (ub[fin] - screen[fin]) + 1e-6 * (1 + np.abs(exact[fin])))


# ---------------------------------------------------------------- k sweep at M = 256 and 128
@pytest.mark.parametrize("name,M,mode,begin,count", [("C4", 256, "sample", 0, 1 << 20), ("C5", 128, "range", 0, 1 << 20)])
@pytest.mark.parametrize("k", [1, 7, 256, 1024])
def test_k_sweep(name, M, mode, begin, count, k):
    o, fit, sp = setup(name, M)
    sp.score_batch(mode=mode, begin=begin, count=count, seed=0, acq="ei", k=k)
    top = sp.topk(k)
    ref, _ = OP.topk(o, fit, mode, begin, count, k, seed=0, acq="ei")
    same_topk(top, ref)


# ---------------------------------------------------------------- sharded exchange on one GPU
@pytest.mark.parametrize("G", [2, 4])
def test_topk_pool_merge_fake_allgather(G):
    from paper_2603_11603_b200.shard import shard_range
    o, fit, _ = setup("C4", 256)
    begin, count, k = 0, 1 << 21, 32
    pools, counts, cuts = [], [], []
    cap = k + max(k, 64)
    for r in range(G):
        _, _, sp = setup("C4", 256)
        lo, n = shard_range(begin, count, r, G)
        sp.score_batch(mode="sample", begin=lo, count=n, seed=0, acq="ei", k=k)
        pool, npool, cut = sp.topk_pool(k, cap)
        pools.append(pool)
        counts.append(npool)
        cuts.append(cut[0])
    merged, cert = A.topk_merge(np.stack(pools), np.array(counts), np.array(cuts), k)
    assert cert
    _, _, sp1 = setup("C4", 256)
    sp1.score_batch(mode="sample", begin=begin, count=count, seed=0, acq="ei", k=k)
    single = sp1.topk(k)
    ref, _ = OP.topk(o, fit, "sample", begin, count, k, seed=0, acq="ei")
    same_topk(merged, ref)
    same_topk(single, ref)


# ---------------------------------------------------------------- ADVICE (round 1)
def test_kappa_xi_validated():
    _, _, sp = setup("C2", 64)
    for kw in (dict(acq="lcb", kappa=-1.0), dict(acq="lcb", kappa=float("nan")), dict(acq="ei", xi=float("inf"))):
        with pytest.raises(A.AutoscoutError):
            sp.score_batch(mode="range", begin=0, count=1000, k=8, **kw)


def test_refit_invalidates_pool_and_mixed_accumulate_rejected():
    o, fit, sp = setup("C2", 64)
    sp.score_batch(mode="range", begin=0, count=5000, acq="ei", k=8)
    with pytest.raises(A.AutoscoutError):       # accumulate with another acquisition
        sp.score_batch(mode="range", begin=5000, count=5000, acq="lcb", k=8, accumulate=True)
    raws, costs = observed(o, 64, 0)
    sp.observe([], [])                          # refit (n = 0): the pool belongs to the old fit
    with pytest.raises(A.AutoscoutError):
        sp.topk(8)
    sp.score_batch(mode="range", begin=0, count=5000, acq="ei", k=8)
    assert len(sp.topk(8)) == 8


def test_list_duplicates_returned_once():
    o, fit, sp = setup("C2", 64)
    pos = np.array([10, 11, 12, 10, 13, 11, 10, 500, 501, 500] * 3, dtype=np.int64)
    d = torch.tensor(pos, device="cuda")
    sp.score_batch(mode="list", begin=0, count=len(pos), acq="ei", k=8, d_positions=d)
    top = sp.topk(8)
    raws = [r for r, _ in top]
    assert len(raws) == len(set(raws))
    rec = OP.score_positions(o, OB.Unranker(o), fit, np.unique(pos), acq="ei")
    same_topk(top, OP._topk_of(rec["raw"], rec["score"], 8))


def test_set_gp_hyper_failure_restores_fit():
    o = oracle_space("C1")
    raws, costs = observed(o, 8, 0)
    sp = A.Space(space_path("C1"), 0)
    sp.observe(raws + raws[:1], costs + costs[:1])     # a duplicated observation: K singular without noise
    before = sp.observe_info()
    with pytest.raises(A.AutoscoutError):
        sp.set_gp_hyper([0.5] * len(o.features), 0.1, 1e-300)
    assert sp.observe_info() == before
    sp.score_batch(mode="range", begin=0, count=o.n_cvi(), acq="ei", k=8)
    assert len(sp.topk(8)) == 8


# ---------------------------------------------------------------- device-resident exchange
@pytest.mark.parametrize("G", [1, 2, 4])
def test_topk_pool_device_merge_device(G):
    """Packed device pools of G handles on disjoint shares, concatenated as all_gather_into_tensor
    would, merged on the device == oracle (no pool passes through host memory)."""
    from paper_2603_11603_b200.shard import shard_range
    o, fit, _ = setup("C4", 256)
    begin, count, k = 0, 1 << 21, 32
    cap = k + max(k, 64)
    bufs, spaces = [], []
    for r in range(G):
        _, _, sp = setup("C4", 256)
        lo, n = shard_range(begin, count, r, G)
        sp.score_batch(mode="sample", begin=lo, count=n, seed=0, acq="ei", k=k)
        bufs.append(sp.topk_pool_device(k, cap))
        spaces.append(sp)
    merged, cert = spaces[0].topk_merge_device(torch.cat(bufs), G, cap, k)
    assert cert
    ref, _ = OP.topk(o, fit, "sample", begin, count, k, seed=0, acq="ei")
    same_topk(merged, ref)


def _two_proc_worker(rank, world, port, out_path):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2603_11603_b200.shard import shard_range
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = oracle_space("C2")
    raws, costs = observed(o, 64, 0)
    sp = A.Space(space_path("C2"), 0)
    sp.observe(raws, costs)
    k, cap = 16, 80
    lo, n = shard_range(0, o.n_cvi(), rank, world)
    sp.score_batch(mode="range", begin=lo, count=n, acq="ei", k=k)
    mine = sp.topk_pool_device(k, cap).cpu()          # gloo moves host tensors; NCCL would not
    gathered = torch.empty(world * mine.numel(), dtype=mine.dtype)
    dist.all_gather_into_tensor(gathered, mine)
    merged, cert = sp.topk_merge_device(gathered.cuda(), world, cap, k)
    if rank == 0:
        np.save(out_path, np.array([[r, s] for r, s in merged] + [[int(cert), 0]], dtype=np.float64))
    dist.destroy_process_group()


def test_two_process_exchange_one_gpu(tmp_path):
    """Two ranks on one GPU: real topk_pool_device output through a real process-group all-gather
    and topk_merge_device == the oracle's top-k of the whole space."""
    import socket
    import torch.multiprocessing as tmp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = str(tmp_path / "merged.npy")
    tmp.spawn(_two_proc_worker, args=(2, port, out), nprocs=2, join=True)
    res = np.load(out)
    assert res[-1, 0] == 1.0
    o, fit, _ = setup("C2", 64)
    ref, _ = OP.topk(o, fit, "range", 0, o.n_cvi(), 16, acq="ei")
    assert [int(r) for r in res[:-1, 0]] == [r for r, _ in ref]
    assert np.allclose(res[:-1, 1], [s for _, s in ref], rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- repeated launches (lag mode)
@pytest.mark.timeout(300)
@pytest.mark.parametrize("name,M,mode,count", [("C5", 128, "range", None), ("C4", 48, "sample", 3_000_000),
                                               ("C4", 256, "sample", 3_000_000)])
def test_repeated_launches_same_result(name, M, mode, count):
    """Five back-to-back scoring passes of the one-hot kernel (lag mode for Mp16 <= 128: two
    accumulators, hand-off of tile t - 1 to the finalize warps): identical certified top-32 every
    time.  Regression for a hand-off that left barrier state behind and deadlocked the NEXT launch."""
    o, fit, sp = setup(name, M)
    count = o.n_cvi() if count is None else count
    first = None
    for _ in range(5):
        sp.score_batch(mode=mode, begin=0, count=count, seed=3, acq="ei", k=32)
        top = sp.topk(32)
        torch.cuda.synchronize()
        if first is None:
            first = top
        else:
            assert top == first


# ---------------------------------------------------------------- asynchronous observe
@pytest.mark.parametrize("name,M,mode,count", [("C4", 256, "sample", 3_000_000), ("C2", 64, "range", None),
                                               ("C5", 128, "range", None)])
def test_async_observe_same_results(name, M, mode, count):
    """set_async_observe: observe() returns before the fit, score_batch generates slice 0 while the
    host thread fits; certified top-k, scores and the fit summary equal the synchronous handle's,
    over repeated observe_clear / observe / score / topk cycles (the bench's e2e loop)."""
    o = oracle_space(name)
    raws, costs = observed(o, M, 0)
    count = o.n_cvi() if count is None else count
    ref = A.Space(space_path(name), 0)
    ref.observe(raws, costs)
    ref.score_batch(mode=mode, begin=0, count=count, seed=1, acq="ei", k=32)
    want = ref.topk(32)
    sp = A.Space(space_path(name), 0)
    sp.set_async_observe(True)
    for _ in range(3):
        sp.observe_clear()
        sp.observe(raws, costs)
        sp.score_batch(mode=mode, begin=0, count=count, seed=1, acq="ei", k=32)
        assert sp.topk(32) == want
        assert sp.observe_info() == ref.observe_info()
    torch.cuda.synchronize()


def test_async_observe_deferred_error():
    """A fit that fails on the worker thread (duplicated observation, sn2 ~ 0: K singular) is
    reported by the next call, once; the handle keeps the previous observed set.  (Asynchronous
    only from 128 observations: C5 with 128 + 1.)"""
    o = oracle_space("C5")
    raws, costs = observed(o, 128, 0)
    sp = A.Space(space_path("C5"), 0)
    sp.set_gp_hyper([0.5] * len(o.features), 0.1, 1e-300)
    sp.observe(raws, costs)
    before = sp.observe_info()
    sp.set_async_observe(True)
    sp.observe(raws[:1], costs[:1])                   # returns: the fit runs on the worker thread
    with pytest.raises(A.AutoscoutError):
        sp.score_batch(mode="range", begin=0, count=1 << 20, acq="ei", k=8)
    assert sp.observe_info() == before
    sp.score_batch(mode="range", begin=0, count=1 << 20, acq="ei", k=8)
    assert len(sp.topk(8)) == 8


def test_async_observe_list_mode_and_slices():
    """Asynchronous observe with the early slice-0 generation: a LIST batch and a SAMPLE batch cut
    into several generation slices (set_slice) give the synchronous handle's certified top-k."""
    o = oracle_space("C4")
    raws, costs = observed(o, 256, 0)
    rng = np.random.default_rng(5)
    pos = np.unique(rng.integers(0, o.n_cvi(), 300_000, dtype=np.int64))
    d_pos = torch.tensor(pos, device="cuda")
    results = []
    for async_on in (False, True):
        sp = A.Space(space_path("C4"), 0)
        sp.set_async_observe(async_on)
        sp.set_slice(1 << 20)                            # 3e6 SAMPLE candidates -> 3 slices
        sp.observe(raws, costs)
        sp.score_batch(mode="list", begin=0, count=len(pos), acq="ei", k=32, d_positions=d_pos)
        top_l = sp.topk(32)
        sp.observe_clear()
        sp.observe(raws, costs)
        sp.score_batch(mode="sample", begin=0, count=3_000_000, seed=9, acq="ei", k=32)
        top_s = sp.topk(32)
        results.append((top_l, top_s))
    torch.cuda.synchronize()
    assert results[0] == results[1]
