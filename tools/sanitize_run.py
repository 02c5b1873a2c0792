"""Small workloads for compute-sanitizer (tools/sanitize.sh): every kernel of the library once.
One-hot tensor-core path (C2 M=64 whole space, C4 M=256 window), 3xTF32 path, SIMT path, mask
kernel, device pool pack / merge, ML-II evidence kernel."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_11603_b200.autoscout import Space  # noqa: E402
from bench import observed_with_library  # noqa: E402

n4 = int(os.environ.get("AS_SAN_N", 1 << 14))
for cfg, M, mode, count, path in [("C2", 64, "range", None, "tc2"), ("C4", 256, "sample", n4, "auto"),
                                  ("C5", 128, "range", n4, "auto"),   # lag mode (two accumulators)
                                  ("C2", 64, "range", 20000, "tc"), ("C1", 16, "range", None, "simt")]:
    sp = Space(os.path.join(ROOT, "spaces", f"{cfg}.json"), 0)
    raws, costs = observed_with_library(sp, M, 0)
    sp.observe(raws, costs)
    sp.set_path(path)
    n = sp.n_cvi if count is None else count
    sc = torch.empty(n, dtype=torch.float32, device="cuda")
    scr = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    sp.score_batch(mode=mode, begin=0, count=n, acq="ei", k=16, d_scores=sc, d_screen=scr)
    top = sp.topk(16)
    pool = sp.topk_pool_device(16, 80)
    merged, cert = sp.topk_merge_device(torch.cat([pool, pool]), 2, 80, 16)
    print(cfg, path, "top1", top[0], "merged", merged[0], cert, flush=True)
    # the bench configuration: no per-candidate outputs (early rejection on), asynchronous observe
    sp.set_async_observe(True)
    sp.observe_clear()
    sp.observe(raws, costs)
    sp.score_batch(mode=mode, begin=0, count=n, acq="ei", k=16)
    assert sp.topk(16) == top
sp = Space(os.path.join(ROOT, "spaces", "C2.json"), 0)
raws, costs = observed_with_library(sp, 64, 0)
sp.observe(raws, costs)
bits = torch.zeros(1 << 12, dtype=torch.int32, device="cuda")
sp.mask_range(0, 1 << 17, bits)
sp.ml2(n_set=8, seed=1, apply=False)
torch.cuda.synchronize()
print("sanitize workload done")
