#!/bin/bash
# Dev A/B builds of libautoscout.so with extra -D flags: tools/exp_build.sh NAME -DFLAG ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
B=paper_2603_11603_b200/_build
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo "$@" -Xcompiler -fPIC,-ffp-contract=off \
  -c paper_2603_11603_b200/csrc/engine.cu -o _exp/engine_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _exp/libautoscout_$name.so _exp/engine_$name.o $B/space.cpp.o -cudart static
echo _exp/libautoscout_$name.so
