"""Builds the native library `libflux_b200.so` in-tree for sm_100a.

The library is the C ABI declared in include/flux_b200.h (host C++ + CUDA
kernels). It is built with nvcc directly (no torch extension machinery): the
product has no torch types at its boundary. `-cudart static` keeps it
independent of whichever libcudart the host process already loaded.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libflux_b200.so")

SOURCES = ["flux_kernels.cu", "flux_api.cpp", "flux_shim.cpp"]
HEADERS = ["flux_internal.hpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra: list[str] | None = None) -> str:
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", "flux_b200.h"), os.path.join(ROOT, "include", "flux", "overlap.hpp")]
    deps.append(os.path.abspath(__file__))
    if not force and not _stale(out, deps):
        return out
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
        "-Xcompiler", "-fvisibility=default", "-cudart", "static",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
        *(extra or []),
        "-o", out + ".tmp",
        *[os.path.join(CSRC, s) for s in SOURCES],
        "-lrt", "-ldl", "-lpthread",
    ]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python -m paper_2406_06858_b200.build [--force] [--variant NAME -DFLAG ...]  (variants: profiling only)
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        name, flags = sys.argv[i + 1], sys.argv[i + 2:]
        os.makedirs(os.path.join(HERE, "variants"), exist_ok=True)
        print(build(force=True, verbose=True, out=os.path.join(HERE, "variants", f"lib_{name}.so"), extra=flags))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
