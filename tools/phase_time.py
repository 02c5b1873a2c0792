"""Dev tool: device-time split (generate / score / merge) of the C4 bench batch per path."""
import sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2603_11603_b200.autoscout import Space
from bench import observed_with_library

sp = Space("spaces/C4.json", 0)
raws, costs = observed_with_library(sp, 256, 0)
sp.observe(raws, costs)
sp.set_timing(True)
for path in sys.argv[1:] or ["tc2", "tc"]:
    sp.set_path(path)
    for i in range(3):
        sp.score_batch(mode="sample", begin=0, count=100_000_000, seed=0, acq="ei", k=32)
        top = sp.topk(32)
        torch.cuda.synchronize()
        k, m = sp.last_kernel_ms()
        g, s = sp.last_phase_ms()
        print(f"{path}: kernels {k:.2f} ms (gen {g:.2f} + score {s:.2f}), merge {m:.3f}, top1 {top[0]}", flush=True)
