mkdir -p gpurun_out
nproc > gpurun_out/host_cpu.txt; lscpu | head -20 >> gpurun_out/host_cpu.txt
ncu --set full --clock-control none --import-source on -k regex:"score_tc2" -c 1 -o gpurun_out/prof_r2a python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_r2a.log 2>&1
ncu -i gpurun_out/prof_r2a.ncu-rep --page source --csv --print-source sass > gpurun_out/r2a_sass.csv 2>&1
ncu -i gpurun_out/prof_r2a.ncu-rep --page raw --csv > gpurun_out/r2a_raw.csv 2>&1
ls -la gpurun_out
