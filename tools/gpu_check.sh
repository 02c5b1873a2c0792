mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/gpu_tests.log
python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/gpu_tests.log
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('STEP', d['ms_per_step'], 'SCORE', r['kernel_ms'], 'GEN', r['gen']['ms'], 'FRAC', r['frac'])" || tail -5 gpurun_out/bench.log
