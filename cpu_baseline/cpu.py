"""ctypes wrapper of cpu_baseline/mpedm_cpu.c (built with gcc -O3 -mavx2 -fopenmp,
-ffp-contract=off so its fp64 neighbour decisions match the oracle's operation order)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpedm_cpu.c")
_LIB = os.path.join(_HERE, "libmpedm_cpu.so")
FLAGS = ["-O3", "-mavx2", "-fopenmp", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.tmp{os.getpid()}"
        subprocess.check_call(["gcc", *FLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i, ip, dp, fp = C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_float)
        _lib.cpu_simplex_all.restype = i
        _lib.cpu_simplex_all.argtypes = [fp, i, i, C.c_long, i, i, i, i, ip, dp, i]
        _lib.cpu_ccm_rows.restype = i
        _lib.cpu_ccm_rows.argtypes = [fp, i, i, C.c_long, ip, i, i, i, i, i, i, dp, i]
    return _lib


def _check(rc, what):
    if rc < 0:
        raise ValueError(f"cpu_baseline {what} failed with code {rc}")


def simplex_all(data, E_max=20, tau=1, s_begin=0, s_end=None, nthreads=0):
    data = np.ascontiguousarray(data, dtype=np.float32)
    L, N = data.shape
    s_end = N if s_end is None else s_end
    optE = np.zeros(s_end - s_begin, np.int32)
    rhoE = np.zeros((s_end - s_begin, E_max), np.float64)
    _check(lib().cpu_simplex_all(data.ctypes.data_as(C.POINTER(C.c_float)), N, L, N, E_max, tau, s_begin, s_end,
                                 optE.ctypes.data_as(C.POINTER(C.c_int)), rhoE.ctypes.data_as(C.POINTER(C.c_double)),
                                 nthreads), "simplex_all")
    return optE, rhoE


def ccm_rows(data, E, tau=1, Tp=1, mode=0, exclude_self=True, lib_begin=0, lib_end=None, nthreads=0):
    data = np.ascontiguousarray(data, dtype=np.float32)
    L, N = data.shape
    E = np.ascontiguousarray(E, dtype=np.int32)
    lib_end = N if lib_end is None else lib_end
    rho = np.zeros((lib_end - lib_begin, N), np.float64)
    _check(lib().cpu_ccm_rows(data.ctypes.data_as(C.POINTER(C.c_float)), N, L, N, E.ctypes.data_as(C.POINTER(C.c_int)),
                              tau, Tp, mode, int(exclude_self), lib_begin, lib_end,
                              rho.ctypes.data_as(C.POINTER(C.c_double)), nthreads), "ccm_rows")
    return rho


def threads() -> int:
    return os.cpu_count() or 1
