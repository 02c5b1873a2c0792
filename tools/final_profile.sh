# Round-2 final measurement set on one B200 (one gpurun call): bench line (with the all-core CPU
# baseline), the reference arm, the ncu launch list of the same command, one ncu --set full capture
# of the two kernels of the step, raw / source pages for the summary.
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"score_tc2|gen_kernel" -c 2 -o gpurun_out/prof_final python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_final.log 2>&1
ncu -i gpurun_out/prof_final.ncu-rep --page raw --csv > gpurun_out/final_raw.csv 2>&1
ncu -i gpurun_out/prof_final.ncu-rep --page source --csv --print-source sass > gpurun_out/final_source.csv 2>&1
ls -la gpurun_out | tail -12
tail -c 700 gpurun_out/final_bench.json; echo; tail -c 500 gpurun_out/final_ref.json
