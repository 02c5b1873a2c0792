#!/bin/bash
# Round-2 experiment loop on the GPU box: quick bench line (no CPU baseline) + tc2 parity subset.
mkdir -p gpurun_out
TAG=${1:-exp}
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{t}_bench.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(t, "ms/step %.3f" % d["ms_per_step"], "score %.3f" % r["kernel_ms"], "gen %.3f" % r["gen"]["ms"],
          "frac %.3f" % r["frac"], "top1", d.get("top1"), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print("bench failed", e); print(open(f"gpurun_out/{t}_bench.err").read()[-3000:])
PY
if [ -z "$NOTEST" ]; then
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tc2 or C4 or C5 or variants" 2>&1 | tail -5
fi
