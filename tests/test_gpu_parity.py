"""GPU parity: the CUDA path through the C-ABI vs the oracle, element by element (-m gpu).

Bars (north_star):
  * raw indices, validity masks, valid counts, top-k raw set and order: bit-exact;
  * simulated cost: |d ln cost| <= 1e-5 (SIM score = -ln cost_sim);
  * posterior mean |d mu| <= 1e-5 max(1,|mu|)  (LCB with kappa=0 gives -mu);
  * posterior variance |d s2| <= 1e-5 sf2      (LCB(kappa=1) - LCB(kappa=0) gives sigma);
  * log EI: |d| <= 1e-5 where z >= -3 and s2 >= 1e-3 sf2, else |d EI| <= 1e-5 sigma_f;
  * refined top-k scores: relative 1e-12.
"""

import json
import math

import numpy as np
import pytest

from brute import enumerate_valid_raw
from conftest import space_path
from oracle import feistel, gp as ogp, run, sim
from parity_util import ei_tolerance_ok, observed, oracle_records, oracle_scores, oracle_space, oracle_topk

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
A = pytest.importorskip("paper_2603_11603_b200.autoscout")

_ORC = {}
_SPACES = {}


def case(name, M, mode="range", begin=0, count=None, seed=0, obs_seed=0, path="auto"):
    """Oracle records (cached per inputs) + a GPU space with the same observed set (cached per path)."""
    key = (name, M, mode, begin, count, seed, obs_seed)
    if key not in _ORC:
        o = oracle_space(name)
        raws, costs = observed(o, M, obs_seed)
        fit = run.observed_fit(o, raws, costs)
        n = o.n_cvi() - begin if count is None else count
        rec = oracle_records(o, fit, mode, begin, n, seed)
        _ORC[key] = (o, fit, rec, (raws, costs), (mode, begin, n, seed))
    o, fit, rec, (raws, costs), batch = _ORC[key]
    skey = (name, M, obs_seed, path)
    if skey not in _SPACES:
        sp = A.Space(space_path(name), 0)
        if M:
            sp.observe(raws, costs)
        sp.set_path(path)
        _SPACES[skey] = sp
    return o, fit, rec, _SPACES[skey], batch


def gpu_run(sp, batch, acq, kappa=None, k=32):
    mode, begin, n, seed = batch
    sc = torch.empty(max(n, 1), dtype=torch.float32, device="cuda")
    rw = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    vc = torch.zeros(1, dtype=torch.int64, device="cuda")
    sp.score_batch(mode=mode, begin=begin, count=n, seed=seed, acq=acq, kappa=kappa, k=k,
                   d_scores=sc, d_raw=rw, d_valid_count=vc)
    top = sp.topk(k)
    torch.cuda.synchronize()
    return sc.cpu().numpy()[:n], rw.cpu().numpy()[:n].astype(np.uint64), int(vc.item()), top


def check_topk(got, ref):
    assert [r for r, _ in got] == [r for r, _ in ref]
    for (_, a), (_, b) in zip(got, ref):
        assert a == pytest.approx(b, rel=1e-12, abs=1e-12)


FULL = [("C1", 16), ("C3", 32), ("P0", 16), ("C2", 64)]


@pytest.mark.parametrize("name,M", FULL)
def test_full_space_sim_mask_raw(name, M):
    o, fit, rec, sp, batch = case(name, M)
    sc, rw, nv, top = gpu_run(sp, batch, "sim")
    assert np.array_equal(rw, rec["raw"])                              # decoded tuples, bit-exact
    assert np.array_equal(np.isfinite(sc), rec["valid"])               # validity mask, bit-exact
    assert nv == int(rec["valid"].sum())
    ref = oracle_scores(o, fit, rec, "sim")
    v = rec["valid"]
    assert np.all(np.abs(sc[v] - ref[v]) <= 1e-5 * np.maximum(1.0, np.abs(ref[v])))
    check_topk(top, oracle_topk(rec, ref, 32))


@pytest.mark.parametrize("path", ["simt", "tc", "tc2"])
@pytest.mark.parametrize("name,M", FULL)
def test_full_space_posterior(name, M, path):
    o, fit, rec, sp, batch = case(name, M, path=path)
    s0, _, _, top0 = gpu_run(sp, batch, "lcb", kappa=0.0)
    s1, _, _, top1 = gpu_run(sp, batch, "lcb", kappa=1.0)
    v = rec["valid"]
    mu_gpu = -s0[v].astype(np.float64)
    mu = rec["mu"][v]
    assert np.all(np.abs(mu_gpu - mu) <= 1e-5 * np.maximum(1.0, np.abs(mu)))
    sig_gpu = s1[v].astype(np.float64) - s0[v].astype(np.float64)
    sf2 = fit.sf2
    assert np.all(np.abs(sig_gpu ** 2 - rec["s2"][v]) <= 1e-5 * sf2 + 4e-7)
    check_topk(top0, oracle_topk(rec, oracle_scores(o, fit, rec, "lcb", kappa=0.0), 32))
    check_topk(top1, oracle_topk(rec, oracle_scores(o, fit, rec, "lcb", kappa=1.0), 32))


@pytest.mark.parametrize("path", ["simt", "tc", "tc2"])
@pytest.mark.parametrize("name,M", FULL)
def test_full_space_ei(name, M, path):
    o, fit, rec, sp, batch = case(name, M, path=path)
    sc, _, _, top = gpu_run(sp, batch, "ei")
    ref = oracle_scores(o, fit, rec, "ei")
    v = rec["valid"]
    ok = ei_tolerance_ok(sc[v].astype(np.float64), ref[v], rec["mu"][v], rec["s2"][v], fit.fstar, fit.sf2)
    assert ok.all(), f"{(~ok).sum()} EI values out of tolerance"
    check_topk(top, oracle_topk(rec, ref, 32))


@pytest.mark.parametrize("name,M,mode,begin,count,seed,path", [
    ("C4", 256, "sample", 0, 1 << 16, 0, "tc"),         # bench shape (M=256), 65,536 sampled candidates
    ("C4", 256, "sample", 0, 1 << 16, 0, "simt"),       # same inputs, SIMT posterior
    ("C4", 256, "sample", 0, 1 << 16, 0, "tc2"),        # same inputs, one-hot r^2 on tensor cores
    ("C4", 65, "range", 100_000_000, 30000, 0, "tc"),   # SIMT-r^2 tensor-core kernel at a ragged M
    ("C4", 64, "sample", 12345, 20000, 7, "auto"),      # M at the 64 boundary (tensor cores)
    ("C4", 65, "range", 100_000_000, 30000, 0, "auto"), # M not a multiple of 16, ragged RANGE window
    ("C5", 128, "range", 1_234_567, 50000, 0, "auto"),  # C5 bench M, RANGE window
    ("C5", 1, "sample", 0, 10000, 3, "auto"),           # M = 1 (SIMT)
    ("C5", 1, "sample", 0, 10000, 3, "tc"),             # M = 1 on tensor cores (one 16-wide chunk)
    ("C5", 1, "sample", 0, 10000, 3, "tc2"),            # M = 1, one-hot r^2 (R2 lookahead limited to 1 chunk)
    ("C5", 20, "sample", 77, 30000, 5, "tc2"),          # 2 chunks per tile: R2 lookahead spans tiles
])
def test_large_space_windows(name, M, mode, begin, count, seed, path):
    o, fit, rec, sp, batch = case(name, M, mode, begin, count, seed, path=path)
    s0, rw, nv, top0 = gpu_run(sp, batch, "lcb", kappa=0.0)
    assert np.array_equal(rw, rec["raw"])
    assert np.array_equal(np.isfinite(s0), rec["valid"]) and nv == int(rec["valid"].sum())
    v = rec["valid"]
    mu = rec["mu"][v]
    assert np.all(np.abs(-s0[v].astype(np.float64) - mu) <= 1e-5 * np.maximum(1.0, np.abs(mu)))
    sc, _, _, top = gpu_run(sp, batch, "ei")
    ref = oracle_scores(o, fit, rec, "ei")
    ok = ei_tolerance_ok(sc[v].astype(np.float64), ref[v], rec["mu"][v], rec["s2"][v], fit.fstar, fit.sf2)
    assert ok.all(), f"{(~ok).sum()} EI values out of tolerance"
    check_topk(top, oracle_topk(rec, ref, 32))


def test_edge_cases():
    o, fit, rec, sp, batch = case("C1", 16)
    # k larger than the number of valid candidates -> every valid one, in order
    sc, _, _, top = gpu_run(sp, batch, "ei", k=1024)
    ref = oracle_scores(o, fit, rec, "ei")
    check_topk(top, oracle_topk(rec, ref, 1024))
    assert len(top) == int(np.isfinite(ref).sum())
    # single candidate; empty batch
    sp.score_batch(mode="range", begin=5, count=1, acq="ei", k=1)
    one = sp.topk(1)
    assert one[0][0] == int(rec["raw"][5])
    sp.score_batch(mode="range", begin=0, count=0, acq="ei", k=4)
    assert sp.topk(4) == []
    # errors
    with pytest.raises(A.AutoscoutError) as e:
        sp.score_batch(mode="range", begin=o.n_cvi() - 3, count=4, acq="ei", k=4)
    assert e.value.status == "AS_ERR_INDEX_RANGE"
    empty = A.Space(space_path("C1"), 0)
    with pytest.raises(A.AutoscoutError) as e:
        empty.score_batch(acq="ei", k=4)
    assert e.value.status == "AS_ERR_NO_OBSERVATIONS"
    with pytest.raises(A.AutoscoutError) as e:
        empty.topk(4)
    assert e.value.status == "AS_ERR_STATE"


def test_accumulate_equals_single_batch():
    o, fit, rec, sp, batch = case("C2", 64)
    _, _, _, top_ref = gpu_run(sp, batch, "ei", k=50)
    n = o.n_cvi()
    cuts = [0, 10007, 40000, n]
    for i in range(3):
        sp.score_batch(mode="range", begin=cuts[i], count=cuts[i + 1] - cuts[i], acq="ei", k=50, accumulate=i > 0)
    top = sp.topk(50)
    assert top == top_ref


def test_prior_only_lcb_and_sim_without_observations():
    o = oracle_space("C3")
    fit = run.observed_fit(o, [], [])
    rec = run.score_batch(o, fit, "range", 0, o.n_cvi(), acq="lcb", kappa=2.0)
    sp = A.Space(space_path("C3"), 0)
    sc, rw, nv, top = gpu_run(sp, ("range", 0, o.n_cvi(), 0), "lcb", kappa=2.0)
    v = rec["valid"]
    assert np.all(np.abs(sc[v] - rec["score"][v]) <= 1e-5 * np.maximum(1, np.abs(rec["score"][v])))
    check_topk(top, run.topk(rec, 32))


@pytest.mark.parametrize("name", ["C1", "C3", "P0", "C2"])
def test_mask_range_full(name):
    o = oracle_space(name)
    with open(space_path(name)) as fh:
        doc = json.load(fh)
    struct = enumerate_valid_raw(doc, o.G)
    _, ok, _ = sim.simulate(o, [o.decode_raw(int(r)) for r in struct])
    valid = struct[ok]
    sp = A.Space(space_path(name), 0)
    n = o.n_raw
    bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    vc = torch.zeros(1, dtype=torch.int64, device="cuda")
    sp.mask_range(0, n, bits, vc)
    torch.cuda.synchronize()
    b = bits.cpu().numpy().view(np.uint32)
    got = np.nonzero(np.unpackbits(b.view(np.uint8), bitorder="little")[:n])[0]
    assert np.array_equal(got, valid)
    assert int(vc.item()) == len(valid)


@pytest.mark.parametrize("name,lo", [("C4", 41_000_000_000), ("C4", 3_000_000_000), ("C5", 600_000_000)])
def test_mask_range_window(name, lo):
    o = oracle_space(name)
    with open(space_path(name)) as fh:
        doc = json.load(fh)
    n = 1 << 21
    struct = enumerate_valid_raw(doc, o.G, window=(lo, lo + n))
    ok = sim.simulate(o, [o.decode_raw(int(r)) for r in struct])[1] if len(struct) else np.zeros(0, bool)
    valid = struct[ok] - lo
    sp = A.Space(space_path(name), 0)
    bits = torch.zeros(n // 32, dtype=torch.int32, device="cuda")
    sp.mask_range(lo, n, bits)
    torch.cuda.synchronize()
    got = np.nonzero(np.unpackbits(bits.cpu().numpy().view(np.uint8), bitorder="little"))[0]
    assert np.array_equal(got, valid)


def test_bench_configuration_sampled():
    """C4 at its full bench size (10^8 sampled candidates, M=256, EI): sampled outputs + top-k."""
    o = oracle_space("C4")
    raws, costs = observed(o, 256, 0)
    fit = run.observed_fit(o, raws, costs)
    sp = A.Space(space_path("C4"), 0)
    sp.observe(raws, costs)
    count = 100_000_000
    sc = torch.empty(count, dtype=torch.float32, device="cuda")
    rw = torch.empty(count, dtype=torch.int64, device="cuda")
    sp.score_batch(mode="sample", begin=0, count=count, seed=0, acq="ei", k=32, d_scores=sc, d_raw=rw)
    top = sp.topk(32)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    js = rng.choice(count, 400, replace=False)
    pi = feistel.Feistel(o.n_cvi(), 0)
    digs = [o.cvi_unrank(pi(int(j))) for j in js]
    rec = run.evaluate(o, digs, fit, acq="ei")
    g_sc = sc[torch.as_tensor(js, device="cuda")].cpu().numpy().astype(np.float64)
    g_rw = rw[torch.as_tensor(js, device="cuda")].cpu().numpy().astype(np.uint64)
    assert np.array_equal(g_rw, rec["raw"])
    v = rec["valid"]
    assert np.array_equal(np.isfinite(g_sc), v)
    ok = ei_tolerance_ok(g_sc[v], rec["score"][v], rec["mu"][v], rec["s2"][v], fit.fstar, fit.sf2)
    assert ok.all()
    # top-k: every returned candidate's refined score equals the oracle's; ordered; and no sampled
    # candidate outside the top-k beats the k-th score
    tr = run.evaluate(o, [o.decode_raw(r) for r, _ in top], fit, acq="ei")
    for (r, s), s_ref in zip(top, tr["score"]):
        assert s == pytest.approx(s_ref, rel=1e-12)
    keys = [(-s, r) for r, s in top]
    assert keys == sorted(keys) and len(top) == 32
    kth = top[-1][1]
    topset = {r for r, _ in top}
    for r, s in zip(rec["raw"][v], rec["score"][v]):
        assert int(r) in topset or s < kth or (s == kth and int(r) > top[-1][0])


def test_native_library_is_the_in_tree_build():
    with open("/proc/self/maps") as fh:
        maps = fh.read()
    assert A.LIB_PATH in maps


# One-hot tensor-core kernel variants the presets do not reach: RBF kernel (KT = 1), four SIMT-side
# features (NH = 4, via the gp.onehot_max_width implementation knob), per-feature lengthscales.
VARIANTS = [
    ("C2", {"kernel": "rbf"}, 64, "range", 0, None),
    ("C2", {"onehot_max_width": 16}, 64, "range", 0, None),
    ("C2", {"onehot_max_width": 0, "kernel": "rbf"}, 80, "range", 0, None),
    ("C5", {"lengthscale": [0.3 + 0.1 * (j % 7) for j in range(16)]}, 128, "range", 2_000_000, 40000),
    ("C4", {"onehot_max_width": 40, "sf2": 0.5, "sn2": 0.01}, 96, "sample", 0, 30000),
    # the one-hot kernel below M = 64 (auto path for large batches): one R2 group,
    # fewer chunks than A-ring stages, ragged Mp16
    ("C4", {}, 48, "sample", 0, 30000),
    ("C1", {}, 16, "range", 0, None),
    ("C3", {}, 32, "range", 0, None),
    ("C2", {}, 17, "range", 0, None),
    ("C2", {"kernel": "rbf"}, 5, "range", 10000, 20000),
]


@pytest.mark.parametrize("base,gp,M,mode,begin,count", VARIANTS)
def test_tc2_variants(base, gp, M, mode, begin, count):
    with open(space_path(base)) as fh:
        doc = json.load(fh)
    doc["gp"].update(gp)
    from oracle import space as S
    o = S.load_space(json.dumps(doc))
    raws, costs = observed(o, M, 3)
    fit = run.observed_fit(o, raws, costs)
    n = o.n_cvi() - begin if count is None else count
    rec = oracle_records(o, fit, mode, begin, n, 5)
    sp = A.Space(doc, 0)
    sp.observe(raws, costs)
    sp.set_path("tc2")
    batch = (mode, begin, n, 5)
    s0, rw, nv, top0 = gpu_run(sp, batch, "lcb", kappa=0.0)
    s1, _, _, _ = gpu_run(sp, batch, "lcb", kappa=1.0)
    v = rec["valid"]
    assert np.array_equal(rw, rec["raw"]) and np.array_equal(np.isfinite(s0), v)
    mu = rec["mu"][v]
    assert np.all(np.abs(-s0[v].astype(np.float64) - mu) <= 1e-5 * np.maximum(1.0, np.abs(mu)))
    sig = s1[v].astype(np.float64) - s0[v].astype(np.float64)
    assert np.all(np.abs(sig ** 2 - rec["s2"][v]) <= 1e-5 * fit.sf2 + 4e-7)
    check_topk(top0, oracle_topk(rec, oracle_scores(o, fit, rec, "lcb", kappa=0.0), 32))
    sc, _, _, top = gpu_run(sp, batch, "ei")
    ref = oracle_scores(o, fit, rec, "ei")
    ok = ei_tolerance_ok(sc[v].astype(np.float64), ref[v], rec["mu"][v], rec["s2"][v], fit.fstar, fit.sf2)
    assert ok.all(), f"{(~ok).sum()} EI values out of tolerance"
    check_topk(top, oracle_topk(rec, ref, 32))


@pytest.mark.parametrize("name,M,mode,count,seed", [("C2", 64, "range", None, 0), ("C4", 256, "sample", 2_000_000, 4),
                                                  ("C4", 48, "sample", 2_000_000, 6), ("C5", 128, "range", None, 0)])
def test_topk_without_per_candidate_outputs(name, M, mode, count, seed):
    """The certified top-k without per-candidate outputs (the bench's call) equals the one with
    d_scores (which also runs the FP64 sensitive-row path), and on C2 the oracle's."""
    o = oracle_space(name)
    raws, costs = observed(o, M, 0)
    sp = A.Space(space_path(name), 0)
    sp.observe(raws, costs)
    n = o.n_cvi() if count is None else count
    sp.score_batch(mode=mode, begin=0, count=n, seed=seed, acq="ei", k=32)
    fast = sp.topk(32)
    sc = torch.empty(n, dtype=torch.float32, device="cuda")
    sp.score_batch(mode=mode, begin=0, count=n, seed=seed, acq="ei", k=32, d_scores=sc)
    exact = sp.topk(32)
    torch.cuda.synchronize()
    assert [r for r, _ in fast] == [r for r, _ in exact]
    for (_, a), (_, b) in zip(fast, exact):
        assert a == b
    if name == "C2":
        fit = run.observed_fit(o, raws, costs)
        rec = run.score_batch(o, fit, "range", 0, n, acq="ei")
        check_topk(fast, run.topk(rec, 32))


def test_slices_do_not_change_results():
    """The one-hot path in many small slices (generate + score + merge per slice, pool accumulated
    across slices) returns the same per-candidate scores and certified top-k as one slice."""
    o = oracle_space("C4")
    raws, costs = observed(o, 256, 0)
    n = 3_000_000
    out = []
    for slice_ in (None, 1 << 20, 777_777):
        sp = A.Space(space_path("C4"), 0)
        sp.observe(raws, costs)
        if slice_:
            sp.set_slice(slice_)
        sc = torch.empty(n, dtype=torch.float32, device="cuda")
        sp.score_batch(mode="sample", begin=0, count=n, seed=2, acq="ei", k=32, d_scores=sc)
        top = sp.topk(32)
        torch.cuda.synchronize()
        out.append((sc.cpu().numpy(), top))
    for sc, top in out[1:]:
        assert np.array_equal(sc, out[0][0])
        assert top == out[0][1]
