# Every preset of SURVEY §8(d) through bench.py on one B200 (whole-space RANGE batches; C4: 1e8 SAMPLE)
mkdir -p gpurun_out
for c in P0 C1 C2 C3 C5 C4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/sweep_$c.json 2> gpurun_out/sweep_$c.err
done
python - <<'PY'
import json
for c in ["P0", "C1", "C2", "C3", "C5", "C4"]:
    try:
        d = json.loads(open(f"gpurun_out/sweep_{c}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(c, "failed", e); continue
    r = d["roofline"]
    print(c, d["config"]["candidates_per_step"], round(d["ms_per_step"], 4), f"{d['value']:.3e}", f"{d['valid_per_s']:.3e}",
          r.get("bound"), r.get("kernel"), round(r.get("frac") or 0, 4), r.get("binding_leg"),
          round(d["e2e"]["ms_per_step"], 3), f"{d['cpu_baseline']['value']:.3e}" if "cpu_baseline" in d else None)
PY
