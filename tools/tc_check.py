"""A/B check of the two posterior paths (SIMT vs tcgen05) on the same inputs -- dev tool."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from parity_util import observed, oracle_space
from paper_2603_11603_b200.autoscout import Space

for name, M, mode, begin, count in [("C1", 16, "range", 0, 176), ("C2", 64, "range", 0, 73176),
                                     ("C4", 256, "sample", 0, 65536), ("C5", 128, "range", 1234567, 50000)]:
    o = oracle_space(name)
    raws, costs = observed(o, M, 0)
    res = {}
    for path in ("simt", "tc", "tc2"):
        sp = Space(f"spaces/{name}.json", 0)
        sp.observe(raws, costs)
        sp.set_path(path)
        sc = torch.empty(count, dtype=torch.float32, device="cuda")
        for acq, kap in (("lcb", 0.0), ("lcb", 1.0), ("ei", None)):
            t0 = time.time()
            sp.score_batch(mode=mode, begin=begin, count=count, acq=acq, kappa=kap, k=32, d_scores=sc)
            top = sp.topk(32)
            torch.cuda.synchronize()
            res[(path, acq, kap)] = (sc.cpu().numpy().copy(), top, time.time() - t0)
    for acq, kap in (("lcb", 0.0), ("lcb", 1.0), ("ei", None)):
        a, ta, _ = res[("simt", acq, kap)]
        for other in ("tc", "tc2"):
            b, tb, _ = res[(other, acq, kap)]
            fin = np.isfinite(a)
            same_mask = np.array_equal(fin, np.isfinite(b))
            d = np.abs(a[fin] - b[fin]).max() if fin.any() else 0
            print(f"{name} M={M} {acq} k={kap}: mask_equal={same_mask} max|simt-{other}|={d:.3e} "
                  f"top_equal={[r for r,_ in ta]==[r for r,_ in tb]}", flush=True)
print("TC CHECK DONE")
