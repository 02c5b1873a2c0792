"""Dev aid: one C5 score_batch + topk step by step with launch counts (lag-mode debugging)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_11603_b200.autoscout import Space

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
M = int(sys.argv[2]) if len(sys.argv) > 2 else None
doc = bench.load_doc(cfg)
b = doc["bench"]
sp = Space(os.path.join(bench.ROOT, "spaces", f"{cfg}.json"), 0)
M = M or b["M"]
raws, costs = bench.observed_with_library(sp, M, 0)
sp.observe(raws, costs)
count = int(b.get("count", sp.n_cvi))
for it in range(3):
    n0 = sp.n_launches()
    t0 = time.time()
    sp.score_batch(mode=b["mode"], begin=0, count=count, seed=0, acq=b["acq"], k=b["k"])
    torch.cuda.synchronize()
    print(it, "score launches", sp.n_launches() - n0, "%.1f ms" % ((time.time() - t0) * 1e3), flush=True)
    n0 = sp.n_launches()
    t0 = time.time()
    top = sp.topk(b["k"], allow_uncertified=True)
    torch.cuda.synchronize()
    print(it, "topk launches", sp.n_launches() - n0, "%.1f ms" % ((time.time() - t0) * 1e3), top[:2], flush=True)
