"""Dev tool: device time of the generate-only work (decode + mask + simulator, SIM acquisition,
no GP) vs the full EI pass on the C4 bench batch."""
import sys, time
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2603_11603_b200.autoscout import Space
from bench import observed_with_library

sp = Space("spaces/C4.json", 0)
raws, costs = observed_with_library(sp, 256, 0)
sp.observe(raws, costs)
sp.set_timing(True)
for acq, path in (("sim", "auto"), ("ei", "tc"), ("ei", "tc2")):
    sp.set_path(path)
    ts = []
    for i in range(4):
        sp.score_batch(mode="sample", begin=0, count=100_000_000, seed=0, acq=acq, k=32)
        torch.cuda.synchronize()
        ts.append(sp.last_kernel_ms()[0])
    print(acq, path, "kernel ms", [round(t, 2) for t in ts], flush=True)
