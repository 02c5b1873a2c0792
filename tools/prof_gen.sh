mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"gen_kernel" -c 1 -o gpurun_out/prof_gen python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_gen.log 2>&1
ncu -i gpurun_out/prof_gen.ncu-rep --page source --csv --print-source sass > gpurun_out/gen_sass.csv 2>&1
ncu -i gpurun_out/prof_gen.ncu-rep --page raw --csv > gpurun_out/gen_raw.csv 2>&1
