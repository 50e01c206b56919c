"""Build helper: compiles the sm_100a CUDA library libgirg.so in-tree with nvcc."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "girg.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("girg_device.cuh", "sample.cuh", "hrg.cuh")] + [
    os.path.join(ROOT, "include", "girg.h")]
LIB = os.path.join(HERE, "libgirg.so")
DEBUG_LIB = os.path.join(HERE, "libgirg_debug.so")  # bounds-checked build (-DGIRG_DEBUG)

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",  # canonical arithmetic: no FMA contraction
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    lib = DEBUG_LIB if debug else LIB
    stale = force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(p) for p in DEPS)
    if stale:
        tmp = lib + f".tmp{os.getpid()}"
        cmd = [nvcc(), *NVCC_FLAGS, *(["-DGIRG_DEBUG"] if debug else []), "-o", tmp, *SOURCES]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
