# C5 and the C4 stress variants (M = 48, 128) on the current build, no CPU baseline
mkdir -p gpurun_out
timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_C5.json 2> gpurun_out/r2_C5.err
timeout 300 python bench.py --observed 48 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_M48.json 2> gpurun_out/r2_M48.err
timeout 300 python bench.py --observed 128 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_M128.json 2> gpurun_out/r2_M128.err
python - <<'PY'
import json
for c in ["C5", "M48", "M128"]:
    try:
        d = json.loads(open(f"gpurun_out/r2_{c}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(c, "failed", e); continue
    r = d["roofline"]
    print(c, round(d["ms_per_step"], 4), f"{d['value']:.3e}", r.get("bound"), round(r.get("frac") or 0, 4), r.get("binding_leg"),
          "score", round(r.get("kernel_ms"), 3), "gen", round(r.get("gen", {}).get("ms", 0), 3), "legs", {k: round(v, 3) for k, v in r.get("legs_ms", {}).items()})
PY
