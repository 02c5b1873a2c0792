"""Dev tool: wall time of a batched ML-II search (NEXT-4) on C4 (M = 256) and C2 (M = 64)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import observed_with_library
from paper_2603_11603_b200.autoscout import Space

for name, M in (("C2", 64), ("C4", 256)):
    sp = Space(f"spaces/{name}.json", 0)
    raws, costs = observed_with_library(sp, M, 0)
    sp.observe(raws, costs)
    sp.ml2(n_set=64, seed=0, apply=False)
    for n in (148, 1024):
        torch.cuda.synchronize()
        t = time.perf_counter()
        best, lml, idx = sp.ml2(n_set=n, seed=1, apply=False)
        dt = time.perf_counter() - t
        print(f"{name} M={M} n_set={n}: {dt * 1e3:.1f} ms  ({n / dt:.0f} settings/s, "
              f"{n * M ** 3 / 3 / dt / 1e12:.2f} TFLOP/s FP64 Cholesky-equivalent) best lml {lml:.3f} @ {idx}")
