"""Multi-GPU causal map: one process per GPU, torch.distributed (NCCL) for plumbing only.

Partitioning (the paper's inter-node scheme P:535-551 with static blocks):
  * every rank holds the full L x N dataset in HBM;
  * phase 1: series are split into contiguous blocks, one per rank -> optE shard;
  * the ONE data-path exchange: all-gather of optE (N int32) -- the paper's "master
    broadcasts optE to all workers" -- since phase 2 on every rank needs the
    E of every target;
  * phase 2: library rows are split into contiguous blocks -> rho rows [rows, N];
  * result assembly: gather of the rho row blocks to rank 0 (replaces the per-element HDF5
    writes of P:553-563).
The kernels are deterministic and each rho[i, j] is computed identically whichever rank
owns row i, so the map is byte-identical at any world size.

`run` takes the phase functions as arguments so the sharding/collective logic can be
tested on CPU with the gloo backend (tests/test_distributed_cpu.py).
"""
from __future__ import annotations

from typing import Callable, Optional

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


def gather_rows(local: torch.Tensor, N: int, dst: int = 0, group=None) -> Optional[torch.Tensor]:
    """Gather rho row blocks [rows_r, N] to rank dst -> [N, N] there (None elsewhere)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-N // world)
    buf = torch.full((per, N), float("nan"), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    if rank == dst:
        gl = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, gl, dst=dst, group=group)
        rows = []
        for r in range(world):
            b, e = shard(N, r, world)
            rows.append(gl[r][: e - b])
        return torch.cat(rows)
    dist.gather(buf, None, dst=dst, group=group)
    return None


def run(data: torch.Tensor, E_max: int, tau: int, Tp: int, mode, exclude_self: bool,
        simplex_fn: Callable, ccm_fn: Callable, gather: bool = True, group=None, timers: Optional[dict] = None):
    """Sharded causal map. simplex_fn(data, E_max, tau, s_begin, s_end) -> optE shard;
    ccm_fn(data, E, tau, Tp, mode, exclude_self, lib_begin, lib_end) -> rho rows.
    Returns (E[N], rho rows of this rank, full rho on rank 0 if gather else None)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N = data.shape[1]
    s0, s1 = shard(N, rank, world)
    optE_local = simplex_fn(data, E_max, tau, s0, s1)
    E = all_gather_E(optE_local, N, group)
    l0, l1 = shard(N, rank, world)
    rows = ccm_fn(data, E, tau, Tp, mode, exclude_self, l0, l1)
    full = gather_rows(rows, N, 0, group) if gather else None
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
    cuda = data.is_cuda
    side = torch.cuda.Stream(device=data.device) if (cuda and rank == 0) else None
    # chunk c of rank r: rows [b_r + c * step_r, ...) of its block [b_r, e_r)
    # (chunks are whole multiples of the kernels' 256-library block, so none runs a partial block
    # except at the end of a rank's rows)
    blocks = [shard(N, r, world) for r in range(world)]
    def step_of(rows):
        want = -(-rows // nchunk)                   # ceil(rows / nchunk)
        return max(1, -(-want // align) * align)    # rounded up to a multiple of align
    steps = [step_of(e - b) for b, e in blocks]
    nchunk = max(-(-(e - b) // st) for (b, e), st in zip(blocks, steps))
    per = max(steps)
    bufs = None
    for c in range(nchunk):
        b, e = blocks[rank]
        r0, r1 = min(e, b + c * steps[rank]), min(e, b + (c + 1) * steps[rank])
        buf = torch.empty((per, N), dtype=torch.float32, device=data.device)
        if r1 > r0:
            buf[: r1 - r0] = ccm_fn(data, E, tau, Tp, mode, exclude_self, r0, r1)
        if rank == 0:
            gl = [torch.empty_like(buf) for _ in range(world)]
            dist.gather(buf, gl, dst=0, group=group)
            if side is not None:
                side.wait_stream(torch.cuda.current_stream(data.device))
            ctx = torch.cuda.stream(side) if side is not None else _nullctx()
            with ctx:
                for r in range(world):
                    rb, re = blocks[r]
                    q0, q1 = min(re, rb + c * steps[r]), min(re, rb + (c + 1) * steps[r])
                    if q1 > q0:
                        rho_host[q0:q1].copy_(gl[r][: q1 - q0], non_blocking=side is not None)
                        if side is not None:
                            gl[r].record_stream(side)
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


def libccm_phase_fns():
    """The production phase functions (libccm CUDA path)."""
    from . import libccm

    def simplex_fn(data, E_max, tau, s0, s1):
        return libccm.simplex_optimal_E(data, E_max, tau, s0, s1)

    def ccm_fn(data, E, tau, Tp, mode, excl, l0, l1):
        return libccm.ccm_all_pairs(data, E, tau, Tp, mode, excl, l0, l1)

    return simplex_fn, ccm_fn


def causal_map_distributed_to_host(data: torch.Tensor, rho_host: Optional[torch.Tensor], E_max: int = 20, tau: int = 1,
                                   Tp: int = 1, mode="target", exclude_self: bool = True, nchunk: int = 4, group=None):
    """Production entry with the map delivered to (page-locked) host memory on rank 0."""
    sf, cf = libccm_phase_fns()
    return run_to_host(data, E_max, tau, Tp, mode, exclude_self, sf, cf, rho_host, nchunk, group)


def causal_map_distributed(data: torch.Tensor, E_max: int = 20, tau: int = 1, Tp: int = 1, mode="target",
                           exclude_self: bool = True, gather: bool = True, group=None):
    """Production entry: every rank passes the full dataset on its own GPU."""
    sf, cf = libccm_phase_fns()
    return run(data, E_max, tau, Tp, mode, exclude_self, sf, cf, gather, group)
