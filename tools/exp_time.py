"""Dev tool: score_batch kernel-time split only (no topk), for A/B builds (AUTOSCOUT_LIB)."""
import sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2603_11603_b200.autoscout import Space
from bench import observed_with_library

sp = Space("spaces/C4.json", 0)
raws, costs = observed_with_library(sp, 256, 0)
sp.observe(raws, costs)
sp.set_timing(True)
sp.set_path(sys.argv[1] if len(sys.argv) > 1 else "tc2")
for i in range(3):
    sp.score_batch(mode="sample", begin=0, count=100_000_000, seed=0, acq="ei", k=32)
    torch.cuda.synchronize()
    g, s = sp.last_phase_ms()
print(f"gen {g:.2f} score {s:.2f}", flush=True)
