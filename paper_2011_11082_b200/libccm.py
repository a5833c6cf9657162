"""Thin Python binding of libccm (include/libccm.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libccm.so; this module converts
torch tensors to device pointers, passes torch's current CUDA stream, owns the workspace
and raises on a non-OK status. There is no CPU fallback: if libccm.so is missing or the
device is not a B200 the calls raise.

Names follow the C ABI (PAPER.md problem statement P:316-317):
  embed_knn(series, E, tau, Tp)              -> idx, dist, w          (edm_embed_knn)
  simplex_optimal_E(data, E_max, tau)        -> optE[, rhoE]          (edm_simplex_optimal_E)
  ccm_all_pairs(data, E, tau, Tp, mode)      -> rho rows              (edm_ccm_all_pairs)
  causal_map_host(host array, ...)           -> optE, rho (numpy)     (edm_causal_map_host)
  ccm_tables(data, E, Eq, ...)               -> idx, dist, w          (edm_ccm_tables, table readback)

Workspaces are cached per (kind, device, stream): calls on different CUDA streams never
share scratch memory (the C ABI is reentrant on distinct streams and workspaces).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

from . import build as _build

EDM_OK, EDM_EINVAL, EDM_ETOOSHORT, EDM_EWORKSPACE, EDM_ECUDA, EDM_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
EDM_E_TARGET, EDM_E_LIBRARY = 0, 1
EDM_LOOKUP_U16 = 0x100  # OR-ed into mode: 16-bit lookup targets (include/libccm.h)
E_CAP = 20

EXPORTS = ("edm_embed_knn", "edm_simplex_optimal_E", "edm_ccm_all_pairs", "edm_workspace_bytes",
           "edm_causal_map_host", "edm_last_error", "edm_version", "edm_profile_begin", "edm_profile_end",
           "edm_ccm_lagged", "edm_ccm_lagged_workspace_bytes", "edm_ccm_convergence",
           "edm_ccm_convergence_workspace_bytes", "edm_ccm_tables", "edm_ccm_tables_workspace_bytes", "edm_ccm_rows",
           "edm_release_cached_memory")
PROF_KINDS = ("prep", "simplex_knn", "simplex_rho", "ccm_knn", "lookup", "other")


class EdmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libccm status {status}: {msg}")
        self.status = status


class edm_dataset(C.Structure):
    _fields_ = [("data", C.c_void_p), ("N", C.c_int32), ("L", C.c_int32), ("ld", C.c_int64)]


_lib = None


def load(path: Optional[str] = None):
    """Load libccm.so (built in-tree by build.py). Raises if it is missing: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("LIBCCM_PATH") or _build.LIB
    if not os.path.exists(path):
        raise ImportError(f"libccm.so not found at {path}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    i32, vp, sz = C.c_int32, C.c_void_p, C.c_size_t
    lib.edm_embed_knn.restype = i32
    lib.edm_embed_knn.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp]
    lib.edm_simplex_optimal_E.restype = i32
    lib.edm_simplex_optimal_E.argtypes = [edm_dataset, i32, i32, i32, i32, vp, vp, vp, sz, vp]
    lib.edm_ccm_all_pairs.restype = i32
    lib.edm_ccm_all_pairs.argtypes = [edm_dataset, vp, i32, i32, i32, i32, i32, i32, vp, vp, sz, vp]
    lib.edm_workspace_bytes.restype = sz
    lib.edm_workspace_bytes.argtypes = [i32, i32, i32, i32, i32, i32]
    lib.edm_causal_map_host.restype = i32
    lib.edm_causal_map_host.argtypes = [vp, i32, i32, i32, i32, i32, i32, i32, vp, vp, vp]
    lib.edm_last_error.restype = C.c_char_p
    lib.edm_last_error.argtypes = []
    lib.edm_version.restype = C.c_char_p
    lib.edm_version.argtypes = []
    lib.edm_ccm_lagged.restype = i32
    lib.edm_ccm_lagged.argtypes = [edm_dataset, vp, i32, i32, i32, i32, i32, i32, i32, vp, vp, sz, vp]
    lib.edm_ccm_lagged_workspace_bytes.restype = sz
    lib.edm_ccm_lagged_workspace_bytes.argtypes = [i32, i32, i32, i32, i32]
    lib.edm_ccm_convergence.restype = i32
    lib.edm_ccm_convergence.argtypes = [edm_dataset, vp, i32, i32, i32, i32, vp, i32, vp, i32, i32, i32, vp, vp, vp,
                                        sz, vp]
    lib.edm_ccm_convergence_workspace_bytes.restype = sz
    lib.edm_ccm_convergence_workspace_bytes.argtypes = [i32, i32, i32, i32, i32, i32]
    lib.edm_release_cached_memory.restype = i32
    lib.edm_release_cached_memory.argtypes = []
    lib.edm_ccm_rows.restype = i32
    lib.edm_ccm_rows.argtypes = [edm_dataset, vp, i32, i32, i32, i32, vp, i32, vp, vp, sz, vp]
    lib.edm_ccm_tables.restype = i32
    lib.edm_ccm_tables.argtypes = [edm_dataset, vp, i32, i32, i32, i32, i32, i32, vp, i32, i32, i32, vp, vp, vp, vp, sz,
                                   vp]
    lib.edm_ccm_tables_workspace_bytes.restype = sz
    lib.edm_ccm_tables_workspace_bytes.argtypes = [i32, i32, i32, i32, i32]
    lib.edm_profile_begin.restype = i32
    lib.edm_profile_begin.argtypes = []
    lib.edm_profile_end.restype = i32
    lib.edm_profile_end.argtypes = [vp, vp]
    _lib = lib
    return lib


def _check(status: int):
    if status != EDM_OK:
        raise EdmError(status, load().edm_last_error().decode())


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(t: torch.Tensor, dtype, name):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (libccm has no CPU path)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def _dataset(data: torch.Tensor) -> edm_dataset:
    _require_cuda(data, torch.float32, "data")
    if data.dim() != 2 or data.stride(1) != 1:
        raise ValueError("data must be a [L, N] time-major tensor with unit column stride")
    L, N = data.shape
    return edm_dataset(data.data_ptr(), N, L, data.stride(0))


_ws_cache: dict = {}


def _workspace_for(kind, nbytes: int, device) -> torch.Tensor:
    """Scratch of at least nbytes for `kind` on torch's current stream of `device`. Cached per
    (kind, device, stream) and allocated while that stream is current, so a buffer is only ever
    used on the stream the caching allocator associates it with."""
    device = torch.device(device)
    key = (kind, device, torch.cuda.current_stream(device).cuda_stream)
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < nbytes:
        _ws_cache.pop(key, None)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


def workspace(which: int, N: int, L: int, E_max: int, tau: int, Tp: int, device) -> torch.Tensor:
    nbytes = load().edm_workspace_bytes(which, N, L, E_max, tau, Tp)
    if nbytes == 0:
        raise EdmError(EDM_EINVAL, f"bad workspace request which={which} N={N} L={L} E_max={E_max}")
    return _workspace_for(which, nbytes, device)


def release_workspaces():
    """Drop the cached workspaces and the device memory edm_causal_map_host keeps between calls."""
    _ws_cache.clear()
    if _lib is not None:
        _check(_lib.edm_release_cached_memory())


def embed_knn(series: torch.Tensor, E: int, tau: int = 1, Tp: int = 1, exclude_self: bool = True,
              with_weights: bool = True):
    """kNN table of one series at E (phase-2 form): idx int32 [n_E, E+1], dist fp32, w fp32."""
    _require_cuda(series, torch.float32, "series")
    series = series.contiguous()
    L = series.numel()
    n = max(L - (E - 1) * tau - Tp, 1)
    idx = torch.empty((n, E + 1), dtype=torch.int32, device=series.device)
    dist = torch.empty((n, E + 1), dtype=torch.float32, device=series.device)
    w = torch.empty((n, E + 1), dtype=torch.float32, device=series.device) if with_weights else None
    _check(load().edm_embed_knn(series.data_ptr(), L, E, tau, Tp, int(exclude_self), idx.data_ptr(),
                                dist.data_ptr(), w.data_ptr() if w is not None else None, _stream(series.device)))
    return idx, dist, w


def simplex_optimal_E(data: torch.Tensor, E_max: int = 20, tau: int = 1, s_begin: int = 0,
                      s_end: Optional[int] = None, return_rho: bool = False):
    """Phase 1: optimal E of series [s_begin, s_end) -> int32 tensor (and rhoE [n, E_max])."""
    ds = _dataset(data)
    s_end = ds.N if s_end is None else s_end
    n = s_end - s_begin
    optE = torch.empty(max(n, 0), dtype=torch.int32, device=data.device)
    rhoE = torch.empty((max(n, 0), E_max), dtype=torch.float32, device=data.device) if return_rho else None
    ws = workspace(0, ds.N, ds.L, E_max, tau, 1, data.device)
    _check(load().edm_simplex_optimal_E(ds, E_max, tau, s_begin, s_end, optE.data_ptr(),
                                        rhoE.data_ptr() if rhoE is not None else None, ws.data_ptr(), ws.numel(),
                                        _stream(data.device)))
    return (optE, rhoE) if return_rho else optE


def _mode(mode, lookup: str = "fp32") -> int:
    if lookup not in ("fp32", "u16"):
        raise ValueError(f"lookup must be 'fp32' or 'u16', got {lookup!r}")
    flag = EDM_LOOKUP_U16 if lookup == "u16" else 0
    if mode in ("target", EDM_E_TARGET):
        return EDM_E_TARGET | flag
    if mode in ("library", EDM_E_LIBRARY):
        return EDM_E_LIBRARY | flag
    raise ValueError(f"mode must be 'target' or 'library', got {mode!r}")


def ccm_all_pairs(data: torch.Tensor, E: torch.Tensor, tau: int = 1, Tp: int = 1, mode="target",
                  exclude_self: bool = True, lib_begin: int = 0, lib_end: Optional[int] = None,
                  out: Optional[torch.Tensor] = None, lookup: str = "fp32") -> torch.Tensor:
    """Phase 2: rho[i - lib_begin, j] for library rows [lib_begin, lib_end) and all targets j.
    lookup="u16": the opt-in 16-bit lookup targets (EDM_LOOKUP_U16, include/libccm.h)."""
    ds = _dataset(data)
    _require_cuda(E, torch.int32, "E")
    E = E.contiguous()
    if E.numel() != ds.N:
        raise ValueError("E must have N entries")
    lib_end = ds.N if lib_end is None else lib_end
    rows = lib_end - lib_begin
    if out is None:
        out = torch.empty((max(rows, 0), ds.N), dtype=torch.float32, device=data.device)
    else:
        _require_cuda(out, torch.float32, "out")
        if not out.is_contiguous() or out.numel() < rows * ds.N:
            raise ValueError("out must be contiguous with at least rows*N elements")
    ws = workspace(1, ds.N, ds.L, E_CAP, tau, Tp, data.device)
    _check(load().edm_ccm_all_pairs(ds, E.data_ptr(), tau, Tp, _mode(mode, lookup), int(exclude_self), lib_begin, lib_end,
                                    out.data_ptr(), ws.data_ptr(), ws.numel(), _stream(data.device)))
    return out


def ccm_rows(data: torch.Tensor, E: torch.Tensor, lib_list, tau: int = 1, Tp: int = 1, mode="target",
             exclude_self: bool = True, out: Optional[torch.Tensor] = None, lookup: str = "fp32") -> torch.Tensor:
    """Phase 2 for a list of library rows (edm_ccm_rows): rho[r, j] for library lib_list[r]."""
    ds = _dataset(data)
    _require_cuda(E, torch.int32, "E")
    E = E.contiguous()
    if E.numel() != ds.N:
        raise ValueError("E must have N entries")
    lst = np.ascontiguousarray(np.asarray(lib_list, dtype=np.int32).ravel())
    rows = lst.size
    if out is None:
        out = torch.empty((rows, ds.N), dtype=torch.float32, device=data.device)
    elif not out.is_contiguous() or out.numel() < rows * ds.N or out.dtype != torch.float32:
        raise ValueError("out must be a contiguous float32 tensor with at least rows*N elements")
    ws = workspace(1, ds.N, ds.L, E_CAP, tau, Tp, data.device)
    _check(load().edm_ccm_rows(ds, E.data_ptr(), tau, Tp, _mode(mode, lookup), int(exclude_self), lst.ctypes.data if rows else None,
                               rows, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream(data.device)))
    return out


def ccm_lagged(data: torch.Tensor, E: torch.Tensor, tau: int = 1, lag_min: int = -2, lag_max: int = 2,
               mode="target", exclude_self: bool = True, lib_begin: int = 0, lib_end: Optional[int] = None,
               out: Optional[torch.Tensor] = None, lookup: str = "fp32") -> torch.Tensor:
    """Time-delay cross mapping (edm_ccm_lagged): rho [rows, nlags, N] for lags lag_min..lag_max
    from one set of kNN tables per library block."""
    ds = _dataset(data)
    _require_cuda(E, torch.int32, "E")
    E = E.contiguous()
    if E.numel() != ds.N:
        raise ValueError("E must have N entries")
    lib_end = ds.N if lib_end is None else lib_end
    rows, nlag = lib_end - lib_begin, lag_max - lag_min + 1
    if out is None:
        out = torch.empty((max(rows, 0), nlag, ds.N), dtype=torch.float32, device=data.device)
    nbytes = load().edm_ccm_lagged_workspace_bytes(ds.N, ds.L, tau, lag_min, lag_max)
    if nbytes == 0:
        raise EdmError(EDM_EINVAL, f"bad lagged workspace request N={ds.N} L={ds.L} lags=[{lag_min},{lag_max}]")
    ws = _workspace_for("lagged", nbytes, data.device)
    _check(load().edm_ccm_lagged(ds, E.data_ptr(), tau, lag_min, lag_max, _mode(mode, lookup), int(exclude_self), lib_begin,
                                 lib_end, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream(data.device)))
    return out


def ccm_convergence(data: torch.Tensor, E: torch.Tensor, lib_sizes, orders, tau: int = 1, Tp: int = 1,
                    mode="target", exclude_self: bool = True, lib_begin: int = 0, lib_end: Optional[int] = None,
                    samples: bool = False):
    """CCM convergence test (edm_ccm_convergence, reading R16): rho [rows, n_sizes, N], the mean
    over the R random library sets of each size; with samples=True also every sample
    [rows, n_sizes, R, N]. lib_sizes: ints; orders: int32 [R, L] permutations of 0..L-1 (host)."""
    ds = _dataset(data)
    _require_cuda(E, torch.int32, "E")
    E = E.contiguous()
    if E.numel() != ds.N:
        raise ValueError("E must have N entries")
    sizes = np.ascontiguousarray(np.asarray(lib_sizes, dtype=np.int32).ravel())
    orders = np.ascontiguousarray(np.atleast_2d(np.asarray(orders, dtype=np.int32)))
    if orders.shape[1] != ds.L:
        raise ValueError("orders must be [R, L]")
    R = orders.shape[0]
    lib_end = ds.N if lib_end is None else lib_end
    rows = max(lib_end - lib_begin, 0)
    out = torch.empty((rows, len(sizes), ds.N), dtype=torch.float32, device=data.device)
    smp = torch.empty((rows, len(sizes), R, ds.N), dtype=torch.float32, device=data.device) if samples else None
    nbytes = load().edm_ccm_convergence_workspace_bytes(ds.N, ds.L, tau, Tp, len(sizes), R)
    if nbytes == 0:
        raise EdmError(EDM_EINVAL, f"bad convergence workspace request N={ds.N} L={ds.L} sizes={len(sizes)} R={R}")
    ws = _workspace_for("convergence", nbytes, data.device)
    _check(load().edm_ccm_convergence(ds, E.data_ptr(), tau, Tp, _mode(mode), int(exclude_self),
                                      sizes.ctypes.data, len(sizes), orders.ctypes.data, R, lib_begin, lib_end,
                                      out.data_ptr(), smp.data_ptr() if samples else None, ws.data_ptr(), ws.numel(),
                                      _stream(data.device)))
    return (out, smp) if samples else out


def ccm_tables(data: torch.Tensor, E: torch.Tensor, Eq: int, tau: int = 1, lag_min: int = 1,
               lag_max: Optional[int] = None, mode="target", exclude_self: bool = True, lib_begin: int = 0,
               lib_end: Optional[int] = None, lib_size: int = 0, order=None, with_dist: bool = True,
               with_weights: bool = True):
    """Phase-2 table readback (edm_ccm_tables): the tables of dimension Eq exactly as the hot path
    builds them, for library rows [lib_begin, lib_end) -> idx int32 [rows, n, Eq+1], dist, w fp32
    (None unless requested). lag_min = lag_max = Tp is the single-horizon table; order (host int32
    [L]) + lib_size select one convergence-test library set. Library mode: rows of libraries whose
    E differs from Eq are left at -1 / NaN."""
    ds = _dataset(data)
    _require_cuda(E, torch.int32, "E")
    E = E.contiguous()
    if E.numel() != ds.N:
        raise ValueError("E must have N entries")
    lag_max = lag_min if lag_max is None else lag_max
    lib_end = ds.N if lib_end is None else lib_end
    rows = max(lib_end - lib_begin, 0)
    m_lo, m_hi = max(0, -lag_min), max(0, lag_max)
    n = max(ds.L - (Eq - 1) * tau - m_lo - m_hi, 0)
    idx = torch.full((rows, n, Eq + 1), -1, dtype=torch.int32, device=data.device)
    dist = torch.full((rows, n, Eq + 1), float("nan"), dtype=torch.float32, device=data.device) if with_dist else None
    w = torch.full((rows, n, Eq + 1), float("nan"), dtype=torch.float32, device=data.device) if with_weights else None
    ordp = None
    if order is not None:
        order = np.ascontiguousarray(np.asarray(order, dtype=np.int32).ravel())
        if order.size != ds.L:
            raise ValueError("order must hold L labels")
        ordp = order.ctypes.data
    nbytes = load().edm_ccm_tables_workspace_bytes(ds.N, ds.L, tau, lag_min, lag_max)
    if nbytes == 0:
        raise EdmError(EDM_EINVAL, f"bad tables workspace request N={ds.N} L={ds.L} lags=[{lag_min},{lag_max}]")
    ws = _workspace_for("tables", nbytes, data.device)
    _check(load().edm_ccm_tables(ds, E.data_ptr(), tau, lag_min, lag_max, _mode(mode), int(exclude_self), lib_size,
                                 ordp, lib_begin, lib_end, Eq, idx.data_ptr(),
                                 dist.data_ptr() if dist is not None else None, w.data_ptr() if w is not None else None,
                                 ws.data_ptr(), ws.numel(), _stream(data.device)))
    return idx, dist, w


def causal_map(data: torch.Tensor, E_max: int = 20, tau: int = 1, Tp: int = 1, mode="target",
               exclude_self: bool = True, lookup: str = "fp32"):
    """Both phases on one GPU from a device-resident dataset -> (optE, rho [N, N])."""
    optE = simplex_optimal_E(data, E_max, tau)
    rho = ccm_all_pairs(data, optE, tau, Tp, mode, exclude_self, lookup=lookup)
    return optE, rho


def causal_map_host(data: np.ndarray, E_max: int = 20, tau: int = 1, Tp: int = 1, mode="target",
                    exclude_self: bool = True, rho_out: Optional[np.ndarray] = None, with_rhoE: bool = False,
                    lookup: str = "fp32"):
    """End-to-end from host memory through edm_causal_map_host (H2D, both phases, D2H)."""
    data = np.ascontiguousarray(data, dtype=np.float32)
    L, N = data.shape
    optE = np.empty(N, np.int32)
    rho = rho_out if rho_out is not None else np.empty((N, N), np.float32)
    assert rho.dtype == np.float32 and rho.flags.c_contiguous and rho.size >= N * N
    rhoE = np.empty((N, E_max), np.float32) if with_rhoE else None
    _check(load().edm_causal_map_host(data.ctypes.data, N, L, E_max, tau, Tp, _mode(mode, lookup), int(exclude_self),
                                      optE.ctypes.data, rho.ctypes.data, rhoE.ctypes.data if with_rhoE else None))
    return (optE, rho, rhoE) if with_rhoE else (optE, rho)


def profile_begin():
    """Start bracketing every libccm launch on this thread with CUDA events (bench.py)."""
    _check(load().edm_profile_begin())


def profile_end():
    """Stop profiling -> {kind: (device ms summed over launches, launch count)}."""
    ms = (C.c_double * len(PROF_KINDS))()
    n = (C.c_int64 * len(PROF_KINDS))()
    _check(load().edm_profile_end(ms, n))
    return {k: (ms[i], n[i]) for i, k in enumerate(PROF_KINDS)}
