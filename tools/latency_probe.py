"""Dev tool: host-side latency split of a small certified pass (C1, M = 16): score_batch vs topk."""
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import observed_with_library
from paper_2603_11603_b200.autoscout import Space

for name, M in (("C1", 16), ("C2", 64)):
    sp = Space(f"spaces/{name}.json", 0)
    raws, costs = observed_with_library(sp, M, 0)
    sp.observe(raws, costs)
    for _ in range(20):
        sp.score_batch(acq="ei", k=32)
        sp.topk(32)
    torch.cuda.synchronize()
    n = 200
    t_sb = t_tk = 0.0
    for _ in range(n):
        t0 = time.perf_counter()
        sp.score_batch(acq="ei", k=32)
        t1 = time.perf_counter()
        sp.topk(32)
        t2 = time.perf_counter()
        t_sb += t1 - t0
        t_tk += t2 - t1
    print(f"{name}: score_batch {1e6 * t_sb / n:.1f} us (host, async), topk {1e6 * t_tk / n:.1f} us (incl. sync)")
