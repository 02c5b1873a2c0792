#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py.
# Run on a GPU box: bash tools/sanitize.sh  -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  N=16384; [ "$tool" = racecheck ] && N=4096
  AS_SAN_N=$N timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
