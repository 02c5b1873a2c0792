"""Sharding layer on CPU (not gpu): world_size 2 over gloo.

Each rank takes its contiguous share of the batch (shard.shard_range), produces its refined pool
(here from the oracle, standing in for the GPU's topk_pool -- test infrastructure only), then the
product path runs: shard.gather_merge = one torch.distributed.all_gather of the packed pools +
autoscout_topk_merge (host C++).  Both ranks must end with the identical top-k, equal to the
oracle's global top-k, certified.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_pool(o, fit, lo, n, k, cap, acq):
    from oracle import run
    from paper_2603_11603_b200.autoscout import ENTRY_DTYPE, no_cut
    rec = run.score_batch(o, fit, "range", lo, n, acq=acq)
    ent = run.topk(rec, 10 ** 9)                         # every valid local candidate, total order
    pool = np.zeros(cap, dtype=ENTRY_DTYPE)
    m = min(cap, len(ent))
    for i in range(m):
        pool[i] = (ent[i][1], ent[i][0])
    cut = no_cut()
    if len(ent) > cap:
        cut[0] = (ent[cap][1], ent[cap][0])
    return pool, m, cut


def _worker(rank, world, port, name, k, cap, acq, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from oracle import run, space as S
    from paper_2603_11603_b200.shard import gather_merge, shard_range
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = S.load_space(os.path.join(ROOT, "spaces", f"{name}.json"))
    fit = run.observed_fit(o, [], [])
    lo, n = shard_range(0, o.n_cvi(), rank, world)
    pool, m, cut = _local_pool(o, fit, lo, n, k, cap, acq)
    top, cert = gather_merge(pool, m, cut, k)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([(r, s) for r, s in top] + [(int(cert), 0.0)],
                                                             dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,acq,k,cap", [("C3", "sim", 16, 80), ("C1", "lcb", 8, 72), ("C3", "lcb", 40, 104)])
def test_two_rank_gloo_merge(tmp_path, name, acq, k, cap):
    from oracle import run, space as S
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, name, k, cap, acq, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    res = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True) for r in range(2)]
    assert [tuple(x) for x in res[0]] == [tuple(x) for x in res[1]]      # identical on every rank
    top = [(int(r), float(s)) for r, s in res[0][:-1]]
    cert = bool(res[0][-1][0])
    o = S.load_space(os.path.join(ROOT, "spaces", f"{name}.json"))
    fit = run.observed_fit(o, [], [])
    ref = run.topk(run.score_batch(o, fit, "range", 0, o.n_cvi(), acq=acq), k)
    assert top == ref
    assert cert


def test_shard_range_partition():
    from paper_2603_11603_b200.shard import shard_range
    for count in (0, 1, 7, 100, 10 ** 8 + 3):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_range(5, count, r, world) for r in range(world)]
            assert parts[0][0] == 5
            for (lo, n), (lo2, _) in zip(parts, parts[1:]):
                assert lo + n == lo2
            assert sum(n for _, n in parts) == count
            assert max(n for _, n in parts) - min(n for _, n in parts) <= 1


def test_pack_unpack_roundtrip():
    from paper_2603_11603_b200.autoscout import ENTRY_DTYPE
    from paper_2603_11603_b200.shard import pack_pool, unpack_pools
    pool = np.zeros(5, dtype=ENTRY_DTYPE)
    pool["score"] = [3.5, 2.0, -1.0, -np.inf, 0]
    pool["raw"] = [10, 2 ** 40, 7, 0, 0]
    cut = np.zeros(1, dtype=ENTRY_DTYPE)
    cut[0] = (-2.5, 99)
    mat = np.stack([pack_pool(pool, 3, cut), pack_pool(pool, 2, cut)])
    pools, counts, cuts = unpack_pools(mat, 5)
    assert list(counts) == [3, 2]
    assert np.array_equal(pools[0], pool) and cuts[1]["raw"] == 99 and cuts[0]["score"] == -2.5
