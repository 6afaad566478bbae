"""The C++ drop-in header (include/flux/overlap.hpp) compiles against the
reference-style call sites in tests/cpp and links to libflux_b200.so; host
checks run here, the device checks on the GPU."""
import os
import subprocess

import pytest

from paper_2406_06858_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_overlap_shim.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_overlap_shim")


def _build():
    libdir = os.path.dirname(N.LIB_PATH)
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(os.path.getmtime(SRC), os.path.getmtime(N.LIB_PATH)):
        subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
                        "-L", libdir, "-l:libflux_b200.so", f"-Wl,-rpath,{libdir}"], check=True)
    return BIN


def test_shim_builds_and_host_checks_pass():
    out = subprocess.run([_build(), "--host-only"], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_shim_runs_reference_call_sites_on_gpu():
    out = subprocess.run([_build()], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
