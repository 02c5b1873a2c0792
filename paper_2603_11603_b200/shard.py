"""Sharding layer: split one scoring batch across 1/2/4/8 GPUs (one process per GPU) and merge
the per-GPU top-k with ONE all-gather.

The candidate positions [begin, begin+count) are cut into `world` contiguous shares (remainder to
the lowest ranks); each rank scores its share on its own device, refines its pool in FP64 and
exports it with an upper bound ("cut") on every candidate it dropped.

Two exchanges, same result:
  * device-resident (GPU ranks, the bench path): `topk_pool_device` packs the pool in device
    memory, ONE `all_gather_into_tensor` (NCCL over NVLink / NVSwitch) concatenates the ranks'
    buffers, `topk_merge_device` merges and certifies on the device; only the k-entry result is
    read back -- no host bounce of any pool;
  * host arrays (`gather_merge`; gloo in the CPU tests): `topk_pool` to host, `all_gather`, host
    C++ `topk_merge`.
Every rank ends with the identical top-k.
"""

from __future__ import annotations

import numpy as np

from .autoscout import ENTRY_DTYPE, topk_merge


def shard_range(begin, count, rank, world):
    share, rem = divmod(count, world)
    lo = begin + rank * share + min(rank, rem)
    return lo, share + (1 if rank < rem else 0)


def pack_pool(pool, n, cut):
    """-> int64 array [4 + 2*cap]: (n, 0, cut entry (score bits, raw), then (score bits, raw) pairs)."""
    cap = len(pool)
    buf = np.zeros(4 + 2 * cap, dtype=np.int64)
    buf[0] = n
    buf[2:4] = np.ascontiguousarray(cut, dtype=ENTRY_DTYPE).view(np.int64)
    buf[4:] = np.ascontiguousarray(pool, dtype=ENTRY_DTYPE).view(np.int64)
    return buf


def unpack_pools(mat, cap):
    mat = np.asarray(mat, dtype=np.int64).reshape(-1, 4 + 2 * cap)
    counts = mat[:, 0].astype(np.int32)
    cuts = np.ascontiguousarray(mat[:, 2:4]).view(ENTRY_DTYPE).reshape(len(mat))
    pools = np.ascontiguousarray(mat[:, 4:]).view(ENTRY_DTYPE).reshape(len(mat), cap)
    return pools, counts, cuts


def gather_merge(pool, n, cut, k, group=None, device=None):
    """All-gather packed pools (one collective) and merge -> (top-k list, certified)."""
    import torch
    import torch.distributed as dist

    cap = len(pool)
    packed = torch.from_numpy(pack_pool(pool, n, cut))
    if device is not None:
        packed = packed.to(device)
    world = dist.get_world_size(group)
    outs = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(outs, packed, group=group)
    mat = torch.stack(outs).cpu().numpy()
    pools, counts, cuts = unpack_pools(mat, cap)
    return topk_merge(pools, counts, cuts, k)


def score_topk_sharded(space, k, begin, count, rank, world, mode="sample", seed=0, acq="ei", cap=None,
                       group=None, device=None, stream=None):
    """Score this rank's share on its GPU, then merge all ranks' pools.  -> (top-k, certified)."""
    lo, n = shard_range(begin, count, rank, world)
    space.score_batch(mode=mode, begin=lo, count=n, seed=seed, acq=acq, k=k, stream=stream)
    cap = cap or (k + max(k, 64))
    pool, npool, cut = space.topk_pool(k, cap, stream=stream)
    return gather_merge(pool, npool, cut, k, group=group, device=device)


def gather_merge_device(space, k, cap, group=None, stream=None):
    """Device-resident exchange: pack the local pool on the device, one all_gather_into_tensor,
    merge on the device.  -> (top-k list, certified)."""
    import torch
    import torch.distributed as dist

    mine = space.topk_pool_device(k, cap, stream=stream)
    world = dist.get_world_size(group)
    gathered = torch.empty(world * mine.numel(), dtype=mine.dtype, device=mine.device)
    dist.all_gather_into_tensor(gathered, mine, group=group)
    return space.topk_merge_device(gathered, world, cap, k, stream=stream)


def score_topk_sharded_device(space, k, begin, count, rank, world, mode="sample", seed=0, acq="ei", cap=None,
                              group=None, stream=None):
    """GPU ranks: score this rank's share, then the device-resident exchange.  -> (top-k, certified)."""
    lo, n = shard_range(begin, count, rank, world)
    space.score_batch(mode=mode, begin=lo, count=n, seed=seed, acq=acq, k=k, stream=stream)
    cap = cap or (k + max(k, 64))
    return gather_merge_device(space, k, cap, group=group, stream=stream)
