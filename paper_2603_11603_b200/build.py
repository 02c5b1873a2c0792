"""Build libautoscout.so in-tree for sm_100a (nvcc + g++; no torch extension machinery).

    python -m paper_2603_11603_b200.build [--verbose]

Host C++ (space.cpp) is compiled with -ffp-contract=off so the FP64 resource check is
bit-identical to the device path (__dmul_rn/__dadd_rn) and to the oracle (R7).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libautoscout.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES_CU = ["engine.cu"]
SOURCES_CPP = ["space.cpp"]
HEADERS = ["common.cuh", "kernels.cuh", "kernels_gen.cuh", "kernels_lml.cuh", "kernels_pool.cuh", "kernels_tc.cuh", "kernels_tc2.cuh", "tc_ptx.cuh", "host_pool.hpp", "space.hpp", "json.hpp", "../../include/autoscout.h"]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr, flush=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    objs = []
    log = ""
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            log += _run(["g++", "-std=c++17", "-O3", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
                         "-I", "/usr/local/cuda/include", "-c", s, "-o", o], verbose)
        objs.append(o)
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            log += _run([NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xptxas", "-v",
                         "-Xcompiler", "-fPIC,-ffp-contract=off", "-c", s, "-o", o], verbose)
        objs.append(o)
    if force or _stale(LIB, objs):
        log += _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"], verbose)
    if log:
        with open(os.path.join(BUILD, "build.log"), "a") as fh:
            fh.write(log)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
