"""The host GP fit of observe() on the thread pool (csrc/host_pool.hpp): every
element is computed by one task in the sequential loop's order, so L^-1, alpha and ||L^-1||_F are
bit-identical for 1, 3 and 8 host threads (C2, C4 with M = 256; C5 with M = 128)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dump_exe(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("gpfit") / "gpfit_dump")
    src = [os.path.join(ROOT, "tools", "gpfit_dump.cpp"), os.path.join(ROOT, "paper_2603_11603_b200", "csrc", "space.cpp")]
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-pthread",
                        "-I/usr/local/cuda/include", *src, "-o", exe], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("g++ build of the fit driver failed: " + r.stderr[-500:])
    return exe


@pytest.mark.parametrize("name,M", [("C2", 64), ("C4", 256), ("C5", 128)])
def test_fit_bit_identical_across_thread_counts(dump_exe, name, M):
    outs = []
    for n in (1, 3, 8):
        env = dict(os.environ, AS_HOST_THREADS=str(n))
        r = subprocess.run([dump_exe, os.path.join(ROOT, "spaces", f"{name}.json"), str(M)], capture_output=True,
                           env=env, timeout=120)
        assert r.returncode == 0
        assert len(r.stdout) == 8 * (M * M + M + 1)
        outs.append(r.stdout)
    assert outs[0] == outs[1] == outs[2]
