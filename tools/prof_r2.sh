# ncu source-level capture of one score_tc2 launch (one bench step): bash tools/prof_r2.sh TAG [bench args]
mkdir -p gpurun_out
T=${1:-r2a}; shift
ncu --set full --clock-control none --import-source on -k regex:"score_tc2" -c 1 -o gpurun_out/prof_$T python bench.py --steps 1 --warmup 0 --no-cpu-baseline "$@" > gpurun_out/ncu_$T.log 2>&1
ncu -i gpurun_out/prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_sass.csv 2>&1
ncu -i gpurun_out/prof_$T.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>&1
rm -f gpurun_out/prof_$T.ncu-rep
