"""Build libccm.so (the C-ABI library of include/libccm.h) in-tree with nvcc for sm_100a.

No JIT cache, no torch extension: a plain `nvcc -shared` so the .so travels with the repo
snapshot to the GPU box and is the one the tests/bench load (paper_2011_11082_b200/lib/libccm.so).
"""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "lib", "libccm.so")
LIB_CHECKED = os.path.join(PKG, "lib", "libccm_checked.so")  # -DCCM_CHECKS: device bounds checks

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # no fast-math, no FMA contraction: the fp64 distance / forecast / Pearson code relies on
    # separately rounded IEEE ops (explicit fmaf() is still used where contraction is wanted)
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    if force or _stale(lib):
        tmp = f"{lib}.tmp{os.getpid()}"  # per process: concurrent ranks never write the same file
        cmd = ["nvcc", *NVCC_FLAGS, *(["-DCCM_CHECKS"] if checked else []), "-I", INCLUDE, "-I", CSRC, "-o", tmp,
               *sources()]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        os.makedirs(os.path.dirname(lib), exist_ok=True)
        subprocess.check_call(cmd)
        os.replace(tmp, lib)  # atomic
    return lib


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose=True, checked="--checked" in sys.argv))
