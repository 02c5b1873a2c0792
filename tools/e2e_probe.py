"""Dev aid: host-side timeline of one e2e step (observe_clear, observe, score_batch, topk) with and
without the asynchronous observe."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2603_11603_b200.autoscout import Space

sp = Space(os.path.join(bench.ROOT, "spaces", "C4.json"), 0)
raws, costs = bench.observed_with_library(sp, 256, 0)
st = torch.cuda.current_stream()
h_raw = torch.tensor(np.asarray(raws, dtype=np.int64)).pin_memory().numpy().view(np.uint64)
h_cost = torch.tensor(np.asarray(costs, dtype=np.float64)).pin_memory().numpy()
for mode in (False, True, False, True):
    sp.set_async_observe(mode)
    for it in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record(st)
        sp.observe_clear(); t1 = time.perf_counter()
        sp.observe(h_raw, h_cost, stream=st); t2 = time.perf_counter()
        sp.score_batch(mode="sample", begin=0, count=100_000_000, seed=0, acq="ei", k=32, stream=st); t3 = time.perf_counter()
        top = sp.topk(32, stream=st); t4 = time.perf_counter()
        e1.record(st); torch.cuda.synchronize()
        if it == 3:
            print("async" if mode else "sync ", "clear %.2f observe %.2f score_batch %.2f topk %.2f  | gpu e2e %.2f ms" %
                  ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, e0.elapsed_time(e1)), flush=True)
