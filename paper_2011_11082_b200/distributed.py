"""Multi-GPU causal map: one process per GPU, torch.distributed (NCCL) for plumbing only.

Partitioning (the paper's inter-node scheme P:535-551 with static blocks):
  * every rank holds the full L x N dataset in HBM;
  * phase 1: series are split into contiguous blocks, one per rank -> optE shard;
  * the ONE data-path exchange: all-gather of optE (N int32) -- the paper's "master
    broadcasts optE to all workers" -- since phase 2 on every rank needs the
    E of every target;
  * phase 2: library rows are split into contiguous blocks in target mode (uniform cost) and
    dealt round-robin over an E-sorted order in library mode (cost grows with the library's E)
    -> rho rows [rows, N] (assign_rows);
  * result assembly: gather of the rho row blocks to rank 0 (replaces the per-element HDF5
    writes of P:553-563).
The kernels are deterministic and each rho[i, j] is computed identically whichever rank
owns row i, so the map is byte-identical at any world size.

`run` takes the phase functions as arguments so the sharding/collective logic can be
tested on CPU with the gloo backend (tests/test_distributed_cpu.py).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


def shard(n: int, rank: int, world: int):
    """Contiguous block [begin, end) of rank among world (sizes differ by at most 1)."""
    base, rem = divmod(n, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def all_gather_E(local: torch.Tensor, N: int, group=None) -> torch.Tensor:
    """All-gather variable-size optE shards (padded to the largest shard) -> E[N] int32."""
    world = dist.get_world_size(group)
    per = -(-N // world)
    buf = torch.zeros(per, dtype=torch.int32, device=local.device)
    buf[: local.numel()] = local
    out = torch.empty(per * world, dtype=torch.int32, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    parts = []
    for r in range(world):
        b, e = shard(N, r, world)
        parts.append(out[r * per: r * per + (e - b)])
    return torch.cat(parts)


def assign_rows(E, world: int, mode) -> list:
    """Library rows of every rank (phase 2), identical on every rank (computed from E[], no
    exchange). Target mode: contiguous blocks (a library's cost does not depend on its own E:
    every library builds the tables of every E in S). Library mode: the table is built at the
    library's own E, so its cost grows with E_i; rows are sorted by E descending (stable) and dealt
    round-robin, rank r taking positions r, r + world, ..., each list ascending."""
    E = np.asarray(E.cpu() if hasattr(E, "cpu") else E)
    N = E.shape[0]
    if mode in ("library", 1):
        order = np.argsort(-E.astype(np.int64), kind="stable")
        return [np.sort(order[r::world]).astype(np.int32) for r in range(world)]
    return [np.arange(*shard(N, r, world), dtype=np.int32) for r in range(world)]


def _is_range(rows: np.ndarray) -> bool:
    return rows.size == 0 or (rows[-1] - rows[0] + 1 == rows.size and np.all(np.diff(rows) == 1))


def gather_rows(local: torch.Tensor, rows_all: list, N: int, dst: int = 0, group=None) -> Optional[torch.Tensor]:
    """Gather every rank's rho rows (local [len(rows_all[rank]), N]) to rank dst -> the [N, N] map
    there, row i at its library index (None elsewhere)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = max(max(len(r) for r in rows_all), 1)
    buf = torch.full((per, N), float("nan"), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    if rank == dst:
        gl = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, gl, dst=dst, group=group)
        full = torch.empty((N, N), dtype=local.dtype, device=local.device)
        for r in range(world):
            rows = rows_all[r]
            if rows.size:
                full[torch.from_numpy(rows.astype(np.int64)).to(local.device)] = gl[r][: rows.size]
        return full
    dist.gather(buf, None, dst=dst, group=group)
    return None


def run(data: torch.Tensor, E_max: int, tau: int, Tp: int, mode, exclude_self: bool,
        simplex_fn: Callable, ccm_fn: Callable, gather: bool = True, group=None, timers: Optional[dict] = None):
    """Sharded causal map. simplex_fn(data, E_max, tau, s_begin, s_end) -> optE shard;
    ccm_fn(data, E, tau, Tp, mode, exclude_self, rows) -> rho rows of the libraries `rows`
    (an ascending int32 array from assign_rows).
    Returns (E[N], rho rows of this rank, full rho on rank 0 if gather else None)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N = data.shape[1]
    s0, s1 = shard(N, rank, world)
    optE_local = simplex_fn(data, E_max, tau, s0, s1)
    E = all_gather_E(optE_local, N, group)
    rows_all = assign_rows(E, world, mode)
    rows = ccm_fn(data, E, tau, Tp, mode, exclude_self, rows_all[rank])
    full = gather_rows(rows, rows_all, N, 0, group) if gather else None
    return E, rows, full


CHUNK_ALIGN = 256  # libraries per phase-2 block of libccm (CCM_B)


def run_to_host(data: torch.Tensor, E_max: int, tau: int, Tp: int, mode, exclude_self: bool,
                simplex_fn: Callable, ccm_fn: Callable, rho_host: Optional[torch.Tensor], nchunk: int = 4,
                group=None, align: int = CHUNK_ALIGN):
    """Sharded causal map delivered to host memory on rank 0 (rho_host [N, N], page-locked for
    overlap; None on other ranks). Phase 2 runs in nchunk row chunks per rank; after each chunk
    the ranks gather it to rank 0 (NCCL), and rank 0 copies it to rho_host on a side stream while
    every rank computes the next chunk. Returns E[N]."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N = data.shape[1]
    s0, s1 = shard(N, rank, world)
    E = all_gather_E(simplex_fn(data, E_max, tau, s0, s1), N, group)
    rows_all = assign_rows(E, world, mode)
    cuda = data.is_cuda
    side = torch.cuda.Stream(device=data.device) if (cuda and rank == 0) else None
    # chunk c of rank r: positions [c * step_r, (c + 1) * step_r) of its row list (chunks are whole
    # multiples of the kernels' 256-library block, so none runs a partial block except at the end)
    def step_of(rows):
        want = -(-rows // nchunk)                   # ceil(rows / nchunk)
        return max(1, -(-want // align) * align)    # rounded up to a multiple of align
    steps = [step_of(len(r)) for r in rows_all]
    nchunk = max(max(-(-len(r) // st) for r, st in zip(rows_all, steps)), 1)
    per = max(steps)
    bufs = None
    for c in range(nchunk):
        mine = rows_all[rank][c * steps[rank]: (c + 1) * steps[rank]]
        buf = torch.empty((per, N), dtype=torch.float32, device=data.device)
        if mine.size:
            buf[: mine.size] = ccm_fn(data, E, tau, Tp, mode, exclude_self, mine)
        if rank == 0:
            gl = [torch.empty_like(buf) for _ in range(world)]
            dist.gather(buf, gl, dst=0, group=group)
            if side is not None:
                side.wait_stream(torch.cuda.current_stream(data.device))
            ctx = torch.cuda.stream(side) if side is not None else _nullctx()
            with ctx:
                for r in range(world):
                    q = rows_all[r][c * steps[r]: (c + 1) * steps[r]]
                    if not q.size:
                        continue
                    if _is_range(q):
                        rho_host[int(q[0]): int(q[-1]) + 1].copy_(gl[r][: q.size], non_blocking=side is not None)
                        if side is not None:
                            gl[r].record_stream(side)
                    else:  # dealt rows (library mode): scatter on the host
                        rho_host[torch.from_numpy(q.astype(np.int64))] = gl[r][: q.size].cpu()
        else:
            dist.gather(buf, None, dst=0, group=group)
        bufs = buf  # keep the last local buffer alive until the collective has consumed it
    if side is not None:
        side.synchronize()
    del bufs
    return E


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def libccm_phase_fns(lookup: str = "fp32"):
    """The production phase functions (libccm CUDA path); lookup="u16": EDM_LOOKUP_U16."""
    from . import libccm

    def simplex_fn(data, E_max, tau, s0, s1):
        return libccm.simplex_optimal_E(data, E_max, tau, s0, s1)

    def ccm_fn(data, E, tau, Tp, mode, excl, rows):
        if _is_range(rows):  # contiguous block: the range call
            l0 = int(rows[0]) if rows.size else 0
            return libccm.ccm_all_pairs(data, E, tau, Tp, mode, excl, l0, l0 + int(rows.size), lookup=lookup)
        return libccm.ccm_rows(data, E, rows, tau, Tp, mode, excl, lookup=lookup)

    return simplex_fn, ccm_fn


def causal_map_distributed_to_host(data: torch.Tensor, rho_host: Optional[torch.Tensor], E_max: int = 20, tau: int = 1,
                                   Tp: int = 1, mode="target", exclude_self: bool = True, nchunk: int = 4, group=None,
                                   lookup: str = "fp32"):
    """Production entry with the map delivered to (page-locked) host memory on rank 0."""
    sf, cf = libccm_phase_fns(lookup)
    return run_to_host(data, E_max, tau, Tp, mode, exclude_self, sf, cf, rho_host, nchunk, group)


def causal_map_distributed(data: torch.Tensor, E_max: int = 20, tau: int = 1, Tp: int = 1, mode="target",
                           exclude_self: bool = True, gather: bool = True, group=None, lookup: str = "fp32"):
    """Production entry: every rank passes the full dataset on its own GPU."""
    sf, cf = libccm_phase_fns(lookup)
    return run(data, E_max, tau, Tp, mode, exclude_self, sf, cf, gather, group)
