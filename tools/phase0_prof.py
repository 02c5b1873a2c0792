"""Dev tool: one SIM-acquisition pass over the C4 bench batch (generate-only work), for ncu."""
import sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2603_11603_b200.autoscout import Space
from bench import observed_with_library

sp = Space("spaces/C4.json", 0)
raws, costs = observed_with_library(sp, 256, 0)
sp.observe(raws, costs)
sp.score_batch(mode="sample", begin=0, count=100_000_000, seed=0, acq="sim", k=32)
torch.cuda.synchronize()
