# C5 (M = 128) and the C4 stress variants (M = 48, 128) on the default path (quick lines, no CPU leg)
mkdir -p gpurun_out
T=${1:-sm}
python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_C5.json 2> gpurun_out/${T}_C5.err
python bench.py --observed 48 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_M48.json 2> gpurun_out/${T}_M48.err
python bench.py --observed 128 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_M128.json 2> gpurun_out/${T}_M128.err
python - "$T" <<'PY'
import json, sys
t = sys.argv[1]
for c in ["C5", "M48", "M128"]:
    try:
        d = json.loads(open(f"gpurun_out/{t}_{c}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(c, "failed", e, open(f"gpurun_out/{t}_{c}.err").read()[-2000:]); continue
    r = d["roofline"]
    print(c, "ms/step %.3f" % d["ms_per_step"], "score %.3f" % r["kernel_ms"], "gen %.3f" % r.get("gen", {}).get("ms", 0),
          "bound", r["bound"], "frac %.3f" % r["frac"], "legs", {k: round(v, 3) for k, v in r.get("legs_ms", {}).items()},
          "mufu_frac %.3f" % r.get("mufu", {}).get("frac", 0))
PY
