"""ctypes wrapper around oracle/ccm_oracle.c (the fp64 CPU oracle).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product package never imports this module.

Every function cites the PAPER.md passage it follows in ccm_oracle.c; see DESIGN.md
"Oracle" for the readings of silent passages and the pins that check each function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ccm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_EINVAL, OR_ETOOSHORT, OR_ENOMEM = 0, -1, -2, -3
MODE_TARGET, MODE_LIBRARY = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc: -O2 -ffp-contract=off (no FMA contraction, no
    fast-math), so each fp64 add/sub/mul is separately rounded as written."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i, dp, ip, fp = C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_float)
        _lib.oracle_dist2.restype = d
        _lib.oracle_dist2.argtypes = [dp, i, dp, i, i, i]
        _lib.oracle_weights.restype = None
        _lib.oracle_weights.argtypes = [dp, i, dp]
        _lib.oracle_pearson.restype = d
        _lib.oracle_pearson.argtypes = [dp, dp, i]
        _lib.oracle_knn.restype = i
        _lib.oracle_knn.argtypes = [dp, i, i, dp, i, i, i, i, i, ip, dp]
        _lib.oracle_ccm_table.restype = i
        _lib.oracle_ccm_table.argtypes = [dp, i, i, i, i, i, ip, dp, dp]
        _lib.oracle_ccm_subset_table.restype = i
        _lib.oracle_ccm_subset_table.argtypes = [dp, i, i, i, i, i, ip, i, ip, dp]
        _lib.oracle_xmap.restype = d
        _lib.oracle_xmap.argtypes = [ip, dp, i, i, i, dp, i, dp, dp]
        _lib.oracle_simplex_rho_E.restype = d
        _lib.oracle_simplex_rho_E.argtypes = [dp, i, i, i]
        _lib.oracle_simplex.restype = i
        _lib.oracle_simplex.argtypes = [dp, i, i, i, dp, ip]
        _lib.oracle_simplex_all.restype = i
        _lib.oracle_simplex_all.argtypes = [fp, i, i, C.c_long, i, i, i, i, ip, dp, i]
        _lib.oracle_ccm_rows.restype = i
        _lib.oracle_ccm_rows.argtypes = [fp, i, i, C.c_long, ip, i, i, i, i, i, i, i, dp, i]
        _lib.oracle_ccm_lagged_rows.restype = i
        _lib.oracle_ccm_lagged_rows.argtypes = [fp, i, i, C.c_long, ip, i, i, i, i, i, i, i, dp, i]
        _lib.oracle_ccm_convergence_rows.restype = i
        _lib.oracle_ccm_convergence_rows.argtypes = [fp, i, i, C.c_long, ip, i, i, i, i, ip, i, ip, i, i, i, dp, dp,
                                                     i]
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int))


def _f(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


def _check(rc, what):
    if rc < 0:
        raise ValueError(f"oracle {what} failed with code {rc}")
    return rc


def nthreads_default() -> int:
    return os.cpu_count() or 1


def dist2(a, t, b, s, E, tau=1) -> float:
    a, pa = _d(a)
    b, pb = _d(b)
    return lib().oracle_dist2(pa, t, pb, s, E, tau)


def weights(d2) -> np.ndarray:
    d2, p = _d(d2)
    w = np.empty_like(d2)
    lib().oracle_weights(p, len(d2), w.ctypes.data_as(C.POINTER(C.c_double)))
    return w


def pearson(a, b) -> float:
    a, pa = _d(a)
    b, pb = _d(b)
    assert len(a) == len(b)
    return lib().oracle_pearson(pa, pb, len(a))


def knn(a, qlo, qhi, b, clo, chi, E, tau=1, exclude_self=False):
    """Rows t = qlo..qhi of series a against candidates clo..chi of series b (Alg. 3)."""
    a, pa = _d(a)
    b, pb = _d(b)
    rows = max(qhi - qlo + 1, 0)
    idx = np.zeros((rows, E + 1), np.int32)
    d2 = np.zeros((rows, E + 1), np.float64)
    _check(lib().oracle_knn(pa, qlo, qhi, pb, clo, chi, E, tau, int(exclude_self),
                            idx.ctypes.data_as(C.POINTER(C.c_int)), d2.ctypes.data_as(C.POINTER(C.c_double))), "knn")
    return idx, d2


def ccm_table(x, E, tau=1, Tp=1, exclude_self=True):
    """Phase-2 table of one library series (Alg. 2 line 5): idx [n_E, E+1] int32,
    d2 [n_E, E+1] fp64 squared distances, w [n_E, E+1] fp64 weights; row r <-> t=(E-1)tau+r."""
    x, px = _d(x)
    L = len(x)
    n = L - (E - 1) * tau - Tp
    if n < 1:
        raise ValueError("series too short")
    idx = np.zeros((n, E + 1), np.int32)
    d2 = np.zeros((n, E + 1), np.float64)
    w = np.zeros((n, E + 1), np.float64)
    _check(lib().oracle_ccm_table(px, L, E, tau, Tp, int(exclude_self), idx.ctypes.data_as(C.POINTER(C.c_int)),
                                  d2.ctypes.data_as(C.POINTER(C.c_double)), w.ctypes.data_as(C.POINTER(C.c_double))),
           "ccm_table")
    return idx, d2, w


def ccm_subset_table(x, E, perm, l, tau=1, Tp=1, exclude_self=True):
    """Table of one library series over one convergence-test library set (reading R16): the
    first min(l, n_E) labels of perm inside P_E are the candidates. idx [n_E, E+1], d2 fp64."""
    x, px = _d(x)
    perm, pp = _i(perm)
    L = len(x)
    n = L - (E - 1) * tau - Tp
    idx = np.zeros((max(n, 0), E + 1), np.int32)
    d2 = np.zeros((max(n, 0), E + 1), np.float64)
    _check(lib().oracle_ccm_subset_table(px, L, E, tau, Tp, int(exclude_self), pp, l,
                                         idx.ctypes.data_as(C.POINTER(C.c_int)),
                                         d2.ctypes.data_as(C.POINTER(C.c_double))), "ccm_subset_table")
    return idx, d2


def xmap(idx, w, t0, y, Tp=1):
    """Alg. 5 lookup + corrcoef; returns (rho, p, o)."""
    idx, pi = _i(idx)
    w, pw = _d(w)
    y, py = _d(y)
    n, k = idx.shape
    p = np.zeros(n)
    o = np.zeros(n)
    r = lib().oracle_xmap(pi, pw, n, k, t0, py, Tp, p.ctypes.data_as(C.POINTER(C.c_double)),
                          o.ctypes.data_as(C.POINTER(C.c_double)))
    return r, p, o


def simplex_rho_E(x, E, tau=1) -> float:
    x, px = _d(x)
    return lib().oracle_simplex_rho_E(px, len(x), E, tau)


def simplex(x, E_max, tau=1):
    """(optE, rhoE[E_max], all_nan_flag) for one series (Alg. 1 phase 1)."""
    x, px = _d(x)
    rho = np.zeros(E_max)
    flag = C.c_int(0)
    e = lib().oracle_simplex(px, len(x), E_max, tau, rho.ctypes.data_as(C.POINTER(C.c_double)), C.byref(flag))
    return e, rho, bool(flag.value)


def simplex_all(data, E_max, tau=1, s_begin=0, s_end=None, nthreads=None):
    """Phase 1 over series [s_begin, s_end) of a float32 [L, N] dataset -> (optE int32, rhoE fp64)."""
    data, pd = _f(data)
    L, N = data.shape
    s_end = N if s_end is None else s_end
    n = s_end - s_begin
    optE = np.zeros(n, np.int32)
    rhoE = np.zeros((n, E_max), np.float64)
    _check(lib().oracle_simplex_all(pd, N, L, N, E_max, tau, s_begin, s_end, optE.ctypes.data_as(C.POINTER(C.c_int)),
                                    rhoE.ctypes.data_as(C.POINTER(C.c_double)), nthreads or nthreads_default()),
           "simplex_all")
    return optE, rhoE


def ccm_rows(data, E, tau=1, Tp=1, mode=MODE_TARGET, exclude_self=True, lib_begin=0, lib_end=None,
             naive=False, nthreads=None):
    """Phase 2 rows [lib_begin, lib_end) of the causal map -> rho [rows, N] fp64."""
    data, pd = _f(data)
    L, N = data.shape
    E, pe = _i(E)
    lib_end = N if lib_end is None else lib_end
    rho = np.zeros((lib_end - lib_begin, N), np.float64)
    _check(lib().oracle_ccm_rows(pd, N, L, N, pe, tau, Tp, mode, int(exclude_self), lib_begin, lib_end, int(naive),
                                 rho.ctypes.data_as(C.POINTER(C.c_double)), nthreads or nthreads_default()),
           "ccm_rows")
    return rho


def ccm_lagged_rows(data, E, tau=1, lag_min=-2, lag_max=2, mode=MODE_TARGET, exclude_self=True, lib_begin=0,
                    lib_end=None, nthreads=None):
    """Time-delay cross mapping: rho [rows, nlags, N] fp64 for lags
    lag_min..lag_max from one table per (library, E) over the points valid for every lag."""
    data, pd = _f(data)
    L, N = data.shape
    E, pe = _i(E)
    lib_end = N if lib_end is None else lib_end
    nlag = lag_max - lag_min + 1
    rho = np.zeros((lib_end - lib_begin, nlag, N), np.float64)
    _check(lib().oracle_ccm_lagged_rows(pd, N, L, N, pe, tau, lag_min, lag_max, mode, int(exclude_self), lib_begin,
                                        lib_end, rho.ctypes.data_as(C.POINTER(C.c_double)),
                                        nthreads or nthreads_default()), "ccm_lagged_rows")
    return rho


def ccm_convergence_rows(data, E, sizes, perms, tau=1, Tp=1, mode=MODE_TARGET, exclude_self=True, lib_begin=0,
                         lib_end=None, samples=False, nthreads=None):
    """CCM convergence test (reading R16): for every library size
    sizes[q] and random order perms[r] (permutations of 0..L-1), the cross-map skill with the
    library set = the first min(l, n_E) labels of perms[r] inside P_E. Returns the mean over r of
    the non-NaN samples, rho [rows, nsizes, N] fp64, and (samples=True) also every sample
    [rows, nsizes, R, N]."""
    data, pd = _f(data)
    L, N = data.shape
    E, pe = _i(E)
    sizes, psz = _i(sizes)
    perms, pp = _i(np.atleast_2d(perms))
    R = perms.shape[0]
    assert perms.shape[1] == L
    lib_end = N if lib_end is None else lib_end
    rows = lib_end - lib_begin
    mean = np.zeros((rows, len(sizes), N), np.float64)
    smp = np.zeros((rows, len(sizes), R, N), np.float64) if samples else None
    _check(lib().oracle_ccm_convergence_rows(pd, N, L, N, pe, tau, Tp, mode, int(exclude_self), psz, len(sizes), pp, R,
                                             lib_begin, lib_end, mean.ctypes.data_as(C.POINTER(C.c_double)),
                                             smp.ctypes.data_as(C.POINTER(C.c_double)) if samples else None,
                                             nthreads or nthreads_default()), "ccm_convergence_rows")
    return (mean, smp) if samples else mean
