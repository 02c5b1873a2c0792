# A/B of library builds on the small-M configurations: bash tools/ab_small.sh libA libB ...
for v in "$@"; do
  cp _exp/$v.so paper_2603_11603_b200/libautoscout.so
  bash tools/small_m.sh sm_$v 2>&1 | grep -E "C5|M48|M128" | sed "s/^/$v /"
  python bench.py --config C2 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v C2', round(d['ms_per_step'],4), d['roofline'].get('kernel'), round(d['roofline'].get('kernel_ms') or 0,4))"
done
