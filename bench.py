#!/usr/bin/env python
"""Benchmark of the all-pairs CCM hot path (BASELINE.json metric: CCM cross-map pairs/s at
1/2/4/8 B200; end-to-end causal-map seconds).

One step = the whole hot path over the synthetic workload:
phase 1 (optimal E of every series, sharded) -> all-gather of E (NCCL) -> phase 2 (all
N x N cross maps, library rows sharded) -> gather of the rho row blocks to rank 0.
value = N^2 pairs per step / device step time (max over ranks), whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--mode target]
  python bench.py --impl reference ...   # the fp64 oracle on the host cores (bounded sample)

Workload at N=1: c3 = 53,053 series x L=1,450 (the paper's Fish1_Normo size), the
largest BASELINE config quoted "at 1/2/4/8 B200" that fits one GPU (c4 is quoted on 8).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2011_11082_b200 import synth  # noqa: E402

METRIC = "CCM cross-map pairs/sec (end-to-end causal-map seconds in e2e)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="libccm", choices=["libccm", "reference"])
    ap.add_argument("--config", default="c3", choices=list(synth.CONFIGS))
    ap.add_argument("--N", type=int, default=None, help="override N (smaller runs of the same recipe)")
    ap.add_argument("--L", type=int, default=None, help="override L (long-series runs of the same recipe)")
    ap.add_argument("--mode", default="target", choices=["target", "library"])
    ap.add_argument("--lookup", default="fp32", choices=["fp32", "u16"],
                    help="u16: the opt-in 16-bit lookup targets (EDM_LOOKUP_U16, a separate line; the headline is fp32)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=None, help="oracle sample size (library rows)")
    ap.add_argument("--convergence", default=None,
                    help="CCM convergence test (SURVEY 8(f) f2) over comma-separated library sizes, e.g. 50,200,999")
    ap.add_argument("--samples", type=int, default=4, help="random library sets per size (--convergence)")
    ap.add_argument("--lags", default=None, help="time-delay cross mapping over lags A:B (SURVEY 8(f) f1) "
                                                 "instead of the single-horizon map")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks (nvidia-smi sampler)
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ work accounting
def lookup_smem_bytes(E: np.ndarray, L: int, tau: int, Tp: int, mode: str) -> float:
    """Algorithmic shared-memory bytes of the lookup for ALL N x N pairs:
    per pair n_E * (k + 1) fp32 reads (k gathered neighbour values + the observation)."""
    E = E.astype(np.float64)
    n = L - (E - 1) * tau - Tp
    per_target = n * (E + 2) * 4.0
    N = len(E)
    if mode == "target":
        return float(N * per_target.sum())           # every library x every target at E_target
    return float(N * per_target.sum())               # library mode: row i uses E_i for all N targets


# Shared-memory pipe cost of one lookup row per warp (32 targets), in SM clocks: a conflict-free
# 32-lane gather takes 1 clock, a warp-uniform 16-byte table broadcast 2 (tools/shfl_bench.cu on
# this B200 measures 0.90 and 0.48 per clock per SM including its loop overhead,
# profiles/r01_mio_microbench.txt); a row = k gathers + ceil(k/2) broadcasts + 1 observation read.
GATHER_CLK, BCAST16_CLK = 1.0, 2.0


def lookup_pipe_cycles(E: np.ndarray, L: int, tau: int, Tp: int, mode: str) -> float:
    """SM-clock cycles of the whole map's lookup on the shared-memory pipe (model above)."""
    E = E.astype(np.int64)
    n = lambda e: max(L - (e - 1) * tau - Tp, 0)
    row = lambda e: (e + 1) * GATHER_CLK + ((e + 2) // 2) * BCAST16_CLK + GATHER_CLK
    N = len(E)
    if mode == "target":
        cnt = np.bincount(E, minlength=21)
        return float(sum(-(-int(cnt[e]) // 32) * N * n(e) * row(e) for e in range(1, 21) if cnt[e]))
    ntiles = -(-N // 32)
    return float(sum(ntiles * n(int(e)) * row(int(e)) for e in E))


def knn_updates(E: np.ndarray, L: int, tau: int, Tp: int, mode: str, lib_size: int | None = None) -> float:
    """Algorithmic (pair, E) updates of the phase-2 distance pass: for each
    library, every ordered pair (t, s != t) of P_E at every E up to the largest needed E
    (incremental over E); each update is 2 FP32 lane-operations in the sweep (the
    difference and the fused multiply-add). With a library set of size lib_size (convergence
    test) the candidates per query are min(lib_size, n_E)."""
    def per_lib(etop):
        tot = 0.0
        for e in range(1, etop + 1):
            n = L - (e - 1) * tau - Tp
            tot += n * ((n if lib_size is None else min(lib_size, n)) - 1)
        return tot
    if mode == "target":
        return len(E) * per_lib(int(E.max()))
    return float(sum(per_lib(int(e)) for e in E))


def load_onchip():
    """Measured on-chip peaks (tools/onchip_peaks.cu on a B200 of this pool, profiles/onchip_peaks.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "onchip_peaks.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------ oracle (cpu_baseline / reference arm)
# the paper's only number for this metric and workload -- mpEDM on ONE ABCI node
# (4x V100 + 2x Xeon Gold 6148), Fish1_Normo = c3 (53,053 x 1,450), 1,973 s end to end
# = 53,053^2 / 1,973 s pairs/s. Another machine's figure: context, not a target.
PAPER_C3_1NODE_PAIRS_S = 53053.0 ** 2 / 1973.0
PAPER_C3_REF = "PAPER.md:653 mpEDM, 1 ABCI node (4x V100 + 2x Xeon 6148), Fish1_Normo 53,053 x 1,450, 1,973 s"

ORACLE_RATE = 1.0e9  # oracle work units (fp64 pair-dimension updates + lookup terms) per core-second,
                     # calibrated on the c3 cpu_baseline (phase 1 1.26e9, phase 2 0.91e9 per core-s)


def _series_work(L, tau, emax, fast=False):
    """Phase-1 work of one series: the oracle recomputes every E (queries x candidates x E per
    E); the fast implementation does one incremental pass plus one selection per E (2 per E)."""
    llib = (L + 1) // 2
    ltgt = L - llib
    return float(sum(max(ltgt - 1 - (e - 1) * tau, 0) * max(llib - 1 - (e - 1) * tau, 0) * (2 if fast else e)
                     for e in range(1, emax + 1)))


def _row_work(L, tau, Tp, E, mode, i=0, fast=False):
    """Phase-2 work of one library row: tables (oracle: n_E^2 E per distinct E; fast: n^2 per
    dimension up to the largest E plus n^2 per selected E) + N lookups of n_E (E+1) terms."""
    n = lambda e: float(max(L - (e - 1) * int(tau) - Tp, 0))
    sel = np.unique(E) if mode == "target" else np.array([int(E[i])])
    if fast:
        tables = n(1) * n(1) * (int(sel.max()) + len(sel))
    else:
        tables = sum(n(e) * n(e) * e for e in sel)
    if mode == "target":
        lookups = float(np.sum([n(e) * (e + 1) for e in E]))
    else:
        lookups = len(E) * n(int(E[i])) * (int(E[i]) + 1)
    return float(tables + lookups)


def oracle_sample(data, E, mode, tau, Tp, n_lib, n_series, lags=None, conv=None, budget_s=12.0, impl="oracle"):
    """Time the fp64 oracle, as it stands, on a bounded sample of the same workload: phase 1 on
    n_series series and phase 2 on n_lib library rows x all N targets, each sized from the work
    model above to take about budget_s seconds on the host cores. When a single series / row is
    already over budget (long series) the sample shrinks further -- phase 1 to E = 1..E_s, phase 2
    to the targets of one E -- and its time is scaled by the work-model ratio (stated in the
    description). Returns (cross maps/s extrapolated to the whole workload, seconds, cores, desc)."""
    if impl == "oracle":
        from oracle import oracle as O
        rate = ORACLE_RATE
    else:  # the fast host implementation, same interface for these calls
        from cpu_baseline import cpu as O
        rate = 1.5 * ORACLE_RATE
    L, N = data.shape
    cores = os.cpu_count() or 1
    mcode = 0 if mode == "target" else 1
    notes = []
    # ---- phase 1
    fast = impl != "oracle"
    w1 = _series_work(L, tau, 20, fast)
    t0 = time.perf_counter()
    if w1 / rate <= budget_s:
        ns = int(min(n_series, N, max(1, budget_s * cores * rate / w1)))
        O.simplex_all(data, 20, tau, 0, ns, nthreads=cores)
        t1 = time.perf_counter()
        full1 = (t1 - t0) * N / ns
        notes.append(f"phase 1 on {ns} series ({t1 - t0:.1f} s)")
    else:
        es = max([e for e in range(1, 21) if _series_work(L, tau, e, fast) / rate <= budget_s] or [1])
        ns = min(cores, N)
        O.simplex_all(data, es, tau, 0, ns, nthreads=cores)
        t1 = time.perf_counter()
        scale = w1 / _series_work(L, tau, es, fast)
        full1 = (t1 - t0) * scale * N / ns
        notes.append(f"phase 1 on {ns} series at E=1..{es} ({t1 - t0:.1f} s, x{scale:.1f} by work model to E=1..20)")
    # ---- phase 2
    wrow = np.mean([_row_work(L, tau, Tp, E, mode, i, fast) for i in range(min(N, 64))])
    if lags or conv or wrow / rate <= budget_s:
        nl = int(min(n_lib, N, max(1, budget_s * cores * rate / wrow))) if not (lags or conv) else n_lib
        if lags:
            O.ccm_lagged_rows(data, E, tau, lags[0], lags[1], mcode, True, 0, nl, cores)
        elif conv:
            O.ccm_convergence_rows(data, E, conv[0], conv[1], tau, Tp, mcode, True, 0, nl, nthreads=cores)
        else:
            O.ccm_rows(data, E, tau=tau, Tp=Tp, mode=mcode, exclude_self=True, lib_begin=0, lib_end=nl,
                       nthreads=cores)
        t2 = time.perf_counter()
        full2 = (t2 - t1) * N / nl
        notes.append(f"phase 2 on {nl} library rows x {N} targets ({t2 - t1:.1f} s)")
    else:
        # one E only: the libraries and targets whose E is the most common value
        e0 = int(np.bincount(E).argmax())
        cols = np.flatnonzero(E == e0)
        nt = int(max(1, min(len(cols), budget_s * rate / (L * (e0 + 1)) / 4)))
        sub = np.ascontiguousarray(data[:, cols[:max(nt, min(cores, len(cols)))]])
        nl = min(cores, sub.shape[1])
        Esub = np.full(sub.shape[1], e0, np.int32)
        O.ccm_rows(sub, Esub, tau=tau, Tp=Tp, mode=mcode, exclude_self=True, lib_begin=0, lib_end=nl,
                   nthreads=cores)
        t2 = time.perf_counter()
        scale = wrow / _row_work(L, tau, Tp, Esub, mode, 0, fast)
        full2 = (t2 - t1) * scale * N / nl
        notes.append(f"phase 2 on {nl} library rows x {sub.shape[1]} targets at E={e0} ({t2 - t1:.1f} s, "
                     f"x{scale:.1f} by work model to all {N} targets and their E)")
    full = full1 + full2
    desc = (", ".join(notes) + f", {cores} threads; value = cross maps / (extrapolated full-map time {full:.0f} s)")
    nlag = (lags[1] - lags[0] + 1) if lags else (len(conv[0]) * len(conv[1]) if conv else 1)
    return N * N * nlag / full, t2 - t0, cores, desc


# Sample sizes of the oracle timing, shared by the main arm's cpu_baseline and --impl reference
# (the same sampler, the same sizes, the same E source: one number, measured twice).
ORACLE_SAMPLE_LIBS, ORACLE_SAMPLE_SERIES = 128, 256


def oracle_E(config, data, cfg):
    """The E vector the oracle's phase-2 sample uses: the ORACLE's own optimal E of every series
    (tests/golden/<config>_optE_oracle.npz, written by tools/oracle_full_optE.py, which calls only
    oracle/) when it exists for this exact workload; otherwise the oracle's phase 1 on the first
    ORACLE_SAMPLE_SERIES series with the rest drawn (seeded) from that empirical distribution."""
    L, N = data.shape
    path = os.path.join(ROOT, "tests", "golden", f"{config}_optE_oracle.npz")
    if os.path.exists(path):
        z = np.load(path)
        if int(z["N"]) == N and int(z["L"]) == L:
            return z["optE"].astype(np.int32), f"oracle optE of all {N} series ({os.path.relpath(path, ROOT)})"
    from oracle import oracle as O
    ns = min(N, ORACLE_SAMPLE_SERIES)
    Es, _ = O.simplex_all(data, cfg["E_max"], cfg["tau"], 0, ns)
    E_all = np.random.default_rng(synth.SEED_BASE).choice(Es, N).astype(np.int32)
    E_all[:ns] = Es
    return E_all, f"oracle optE of {ns} series, the other {N - ns} drawn from their distribution"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    """--impl reference: the fp64 oracle on the host cores (rank 0 only), same config/metric.
    Each step times the oracle on a bounded sample of the workload (oracle_sample, the sampler of
    the main arm's cpu_baseline); the reported value is the median over steps of the full-map rate
    EXTRAPOLATED from the sample (per-library time x N / threads), labelled as such."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    data = synth.make_config(args.config, N=args.N, L=args.L)
    L, N = data.shape
    E_all, e_src = oracle_E(args.config, data, cfg)
    n_lib = min(N, args.cpu_sample or ORACLE_SAMPLE_LIBS)
    values, secs_each = [], []
    desc, cores = "", 0
    for _ in range(args.steps):  # the oracle has no warm-up state; W is accepted for the contract
        v, secs, cores, desc = oracle_sample(data, E_all, args.mode, cfg["tau"], cfg["Tp"], n_lib,
                                             min(N, ORACLE_SAMPLE_SERIES))
        values.append(v)
        secs_each.append(secs)
    value = float(statistics.median(values))
    sample = f"{desc}; E: {e_src}; median of {args.steps} step(s)"
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * N * N / value,
        "extrapolated": True, "measured_seconds_per_step": secs_each,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {N} series x L={L}, E=1..{cfg['E_max']}, tau={cfg['tau']}, "
                               f"Tp={cfg['Tp']}, mode={args.mode}", "N": N, "L": L},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
                         "extrapolated": True, "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


# ------------------------------------------------------------------ main arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2011_11082_b200 import build, distributed, libccm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 with torchrun")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        dist.init_process_group("gloo", rank=0, world_size=1)
    if rank == 0:
        build.build()  # one compile if the in-tree library is stale; the other ranks wait for it
    dist.barrier()
    libccm.load()

    cfg = synth.CONFIGS[args.config]
    E_max, tau, Tp = cfg["E_max"], cfg["tau"], cfg["Tp"]
    host = synth.make_config(args.config, N=args.N, L=args.L)  # same seed on every rank
    L, N = host.shape
    host_pinned = torch.from_numpy(host).pin_memory()
    data = host_pinned.to(dev, non_blocking=True)          # every GPU holds the full dataset (8(e))
    torch.cuda.synchronize()

    s0, s1 = distributed.shard(N, rank, world)
    l0, l1 = s0, s1
    per = -(-N // world)
    lags = tuple(int(v) for v in args.lags.split(":")) if args.lags else None
    nlag = (lags[1] - lags[0] + 1) if lags else 1
    conv = None
    if args.convergence:
        conv_sizes = [int(v) for v in args.convergence.split(",")]
        conv = (conv_sizes, synth.library_orders(args.samples, L, synth.SEED_BASE + 7))
        nlag = len(conv_sizes) * args.samples  # cross maps per (library, target) pair
    rho_rows = torch.empty((per, nlag, N) if lags else (per, N), dtype=torch.float32, device=dev)
    gather_list = [torch.empty_like(rho_rows) for _ in range(world)] if (rank == 0 and world > 1) else None
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        optE = libccm.simplex_optimal_E(data, E_max, tau, s0, s1)           # S1-S3
        if ev:
            ev[1].record(stream)
        E = distributed.all_gather_E(optE, N) if world > 1 else optE         # S4 (NCCL all-gather)
        if ev:
            ev[2].record(stream)
        if lags:
            libccm.ccm_lagged(data, E, tau, lags[0], lags[1], args.mode, True, l0, l1, out=rho_rows,
                              lookup=args.lookup)  # f1
        elif conv:
            libccm.ccm_convergence(data, E, conv[0], conv[1], tau, Tp, args.mode, True, l0, l1)  # f2
        elif args.mode == "library" and world > 1:
            # library mode: rows dealt round-robin over the E-sorted order
            rows = distributed.assign_rows(E, world, "library")[rank]
            libccm.ccm_rows(data, E, rows, tau, Tp, "library", True, out=rho_rows, lookup=args.lookup)  # S5-S9
        else:
            libccm.ccm_all_pairs(data, E, tau, Tp, args.mode, True, l0, l1, out=rho_rows, lookup=args.lookup)  # S5-S9
        if ev:
            ev[3].record(stream)
        if world > 1:
            dist.gather(rho_rows, gather_list, dst=0)                        # S10 (NCCL)
        if ev:
            ev[4].record(stream)
        return E

    # warm-up (contexts, NCCL communicators, workspaces, first launches; P:770 straggler lesson)
    for _ in range(max(args.warmup, 0)):
        E = step()
    torch.cuda.synchronize()
    E_host = E.cpu().numpy()

    # timed region: K steps bracketed by barrier + synchronize on both sides
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.6)
    dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    libccm.profile_begin()
    t_start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    prof = libccm.profile_end()
    dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_local = t_start.elapsed_time(t_end)
    phases = np.zeros(4)
    for e in evs:
        phases += [e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]), e[3].elapsed_time(e[4])]
    per_rank = [None] * world
    mine = {"rank": rank, "ms": ms_local, "simplex": phases[0] / args.steps, "allgather_E": phases[1] / args.steps,
            "ccm": phases[2] / args.steps, "gather_rho": phases[3] / args.steps,
            "kernels": {k: round(v[0] / args.steps, 1) for k, v in prof.items()}}
    if world > 1:
        dist.all_gather_object(per_rank, mine)
    else:
        per_rank = [mine]
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev if world > 1 else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_per_step = ms_total / args.steps
    pairs = float(N) * N * nlag
    value = pairs / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel (lookup) from live CUDA-event launch times
    lk_ms, lk_n = prof["lookup"]
    kn_ms, kn_n = prof["ccm_knn"]
    rows_frac = (l1 - l0) / N
    if conv:
        # one lookup pass per (size l, sample) over the pairs whose E admits l (l - 1 >= E + 1):
        # N x sum over those E of the per-target bytes (target mode: targets j, library mode: rows i)
        def conv_bytes(l):
            sub = E_host[E_host <= l - 2]
            return lookup_smem_bytes(sub, L, tau, Tp, args.mode) * N / len(sub) if len(sub) else 0.0
        smem_bytes_step = sum(conv_bytes(l) for l in conv[0]) * args.samples * rows_frac
    else:
        smem_bytes_step = lookup_smem_bytes(E_host, L, tau, Tp, args.mode) * rows_frac * nlag
    bytes_per_launch = smem_bytes_step * args.steps / max(lk_n, 1)
    avg_launch_s = lk_ms / max(lk_n, 1) / 1e3
    peaks = load_peaks()
    sm_max_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    smem_peak = nsm * 128.0 * sm_max_mhz * 1e6 / 1e9  # GB/s: 128 B/clk/SM shared-memory crossbar
    achieved = bytes_per_launch / avg_launch_s / 1e9 if lk_n else None
    traffic = load_traffic().get("lookup_dram_bytes_per_launch")
    ntiles_bytes = (N + 32 * 20) * L * 4.0  # target-tile HBM bytes per lookup launch (upper bound on tiles)
    hbm_peak = float(peaks.get("hbm_gbs", 6555.2))
    roofline = {
        "kernel": "lookup_kernel (S9: gather-weighted lookup + fused Pearson)",
        "bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
        "frac": (achieved / smem_peak) if achieved else None, "traffic": traffic,
        "peak_source": f"derived: {nsm} SMs x 128 B/clk x {sm_max_mhz:.0f} MHz (B300_MICROARCH smem crossbar; "
                       "MEASURED_PEAKS.json has no smem figure -- the measured one is peak_measured)",
        "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_launch_s * 1e3, "launches": lk_n,
        "algorithmic_note": ("--lookup u16: algorithmic bytes counted at the fp32 definition (4 B per gathered or "
                             "observed value, SURVEY 8(d)); the 16-bit codes move 2 B each") if args.lookup == "u16" else None,
        "share_of_step": lk_ms / ms_local if ms_local else None,
        "pipe_model": {"frac": (lookup_pipe_cycles(E_host, L, tau, Tp, args.mode) * (0.5 if args.lookup == "u16" else 1.0)
                                * rows_frac * nlag * args.steps /
                                (nsm * sm_max_mhz * 1e6) / (lk_ms / 1e3)) if (lk_n and not conv) else None,
                       "note": "ideal shared-memory-pipe time of this instruction mix (per row: k gathers x 1 clk "
                               "+ ceil(k/2) uniform 16-B table broadcasts x 2 clk + 1 observation x 1 clk, costs from "
                               "tools/shfl_bench.cu) / measured lookup time" + ("; --lookup u16: the same per-row pipe "
                               "cost serves 64 targets (two 16-bit codes per gathered word), so half the fp32 model's "
                               "cycles" if args.lookup == "u16" else "")},
        "hbm_view": {"bound": "hbm", "target_tile_bytes_per_launch": ntiles_bytes,
                     "achieved": ntiles_bytes / avg_launch_s / 1e9 if lk_n else None, "peak": hbm_peak,
                     "frac": (ntiles_bytes / avg_launch_s / 1e9 / hbm_peak) if lk_n else None,
                     "note": "north_star roof: HBM bytes of the staged target tiles (measured copy peak)"},
    }
    if conv:
        def conv_ops(l):
            sub = E_host[E_host <= l - 2]
            if not len(sub):
                return 0.0
            if args.mode == "target":  # every library builds tables up to the largest admitted E
                return knn_updates(sub[:1] * 0 + sub.max(), L, tau, Tp, "target", l) * N
            return knn_updates(sub, L, tau, Tp, "library", l)
        knn_upd = sum(conv_ops(l) for l in conv[0]) * args.samples * rows_frac
    else:
        knn_upd = knn_updates(E_host, L, tau, Tp, args.mode) * rows_frac
    onchip = load_onchip()
    fp32_peak = nsm * 128.0 * sm_max_mhz * 1e6 / 1e12  # T lane-ops/s: 128 FP32 lanes/clk/SM (4 x 32 per SM)
    kn_ach = knn_upd * 2.0 * args.steps / (kn_ms / 1e3) / 1e12 if kn_n else None
    roofline_knn = {
        "kernel": "phase-2 kNN (S6-S8: incremental fp32 distance sweep + exact fp64 selection + fused weights)",
        "bound": "alu", "unit": "T FP32 lane-ops/s",
        "peak_source": f"derived: {nsm} SMs x 128 FP32 lanes/clk x {sm_max_mhz:.0f} MHz (B200_PROFILING unit counts); "
                       "algorithmic = 2 FP32 ops (difference, fused multiply-add) per (pair, E) update",
        "algorithmic_updates_per_step": knn_upd,
        "achieved": kn_ach, "peak": fp32_peak, "frac": (kn_ach / fp32_peak) if kn_ach else None,
        "peak_measured": (onchip["fp32_ffma_lanes_per_clk_sm"] * nsm * sm_max_mhz * 1e6 / 1e12
                          if onchip.get("fp32_ffma_lanes_per_clk_sm") else None),
        "avg_launch_ms": kn_ms / max(kn_n, 1), "launches": kn_n,
        "share_of_step": kn_ms / ms_local if ms_local else None,
    }
    if roofline_knn["peak_measured"] and kn_ach:
        roofline_knn["frac_measured"] = kn_ach / roofline_knn["peak_measured"]
    if onchip.get("smem_bytes_per_clk_sm") and achieved:
        smem_meas = onchip["smem_bytes_per_clk_sm"] * nsm * sm_max_mhz * 1e6 / 1e9
        roofline["peak_measured"] = smem_meas
        roofline["frac_measured"] = achieved / smem_meas
        roofline["peak_measured_source"] = "profiles/onchip_peaks.json (tools/onchip_peaks.cu, best conflict-free LDS)"
    launches = sum(n for _, n in prof.values())
    # the dominant kernel (largest share of the step) carries "roofline"; the other is kept beside it
    knn_traffic = load_traffic().get("ccm_knn_dram_bytes_per_launch")
    roofline_knn["traffic"] = knn_traffic
    if kn_ms > lk_ms:
        roofline_main, roofline_other, other_key = roofline_knn, roofline, "roofline_lookup"
    else:
        roofline_main, roofline_other, other_key = roofline, roofline_knn, "roofline_knn"

    # ---- end to end through the public API: pinned host input -> H2D -> both phases -> D2H of rho
    e2e = None
    if args.e2e_steps > 0 and not lags and not conv:
        Bi = N * L * 4 * world
        Bo = N * N * 4
        if world == 1:
            rho_host = torch.empty((N, N), dtype=torch.float32).pin_memory().numpy()
            host_np = host_pinned.numpy()
            libccm.release_workspaces()
            torch.cuda.empty_cache()
            libccm.causal_map_host(host_np, E_max, tau, Tp, args.mode, True, rho_out=rho_host, lookup=args.lookup)  # warm
            ts = []
            for _ in range(args.e2e_steps):
                t0 = time.perf_counter()
                libccm.causal_map_host(host_np, E_max, tau, Tp, args.mode, True, rho_out=rho_host, lookup=args.lookup)
                ts.append(time.perf_counter() - t0)
            sec = float(np.mean(ts))  # mean over the timed calls, like ms_per_step (total / K)
        else:
            rho_host = torch.empty((N, N), dtype=torch.float32).pin_memory() if rank == 0 else None
            ts = []
            for _ in range(args.e2e_steps):
                dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                d = host_pinned.to(dev, non_blocking=True)
                distributed.causal_map_distributed_to_host(d, rho_host, E_max, tau, Tp, args.mode, True,
                                                           lookup=args.lookup)
                torch.cuda.synchronize()
                el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
                dist.all_reduce(el, op=dist.ReduceOp.MAX)
                ts.append(float(el.item()))
            sec = float(np.mean(ts))
        e2e = {"value": pairs / sec, "unit": "pairs/s", "seconds": sec, "seconds_each": ts, "h2d_bytes_per_step": Bi,
               "d2h_bytes_per_step": Bo, "api": "edm_causal_map_host (C ABI, host buffers)" if world == 1 else
               "distributed.causal_map_distributed_to_host (pinned H2D, chunked NCCL gather + overlapped D2H)"}

    # ---- CPU baseline: the oracle on a bounded sample, rank 0 at N=1 only
    cpu = None
    unit = "(pair, lag)/s" if lags else "(pair, size, sample)/s" if conv else "pairs/s"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_lib = args.cpu_sample or (min(N, ORACLE_SAMPLE_LIBS) if not conv else min(N, max(16, ORACLE_SAMPLE_LIBS // nlag)))
        E_or, e_src = oracle_E(args.config, host, cfg) if (args.N is None and args.L is None) else (E_host, "the run's E")
        v, secs, cores, desc = oracle_sample(host, E_or, args.mode, tau, Tp, n_lib, min(N, ORACLE_SAMPLE_SERIES), lags,
                                             conv)
        cpu = {"value": v, "unit": unit, "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
               "extrapolated": True, "sample": f"{desc}; E: {e_src}"}

    # ---- fast host implementation (the CPU side of the paper's GPU-vs-CPU
    # comparison; bit-identical to the oracle), same bounded-sample method
    cpu_fast = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not lags and not conv:
        v, secs, cores, desc = oracle_sample(host, E_host, args.mode, tau, Tp, N, N, impl="fast")
        cpu_fast = {"value": v, "unit": unit, "cores": cores, "kind": "fast host implementation (cpu_baseline/)",
                    "sample": desc, "gpu_speedup": value / v}

    full_c3 = args.config == "c3" and N == synth.CONFIGS["c3"]["N"] and L == synth.CONFIGS["c3"]["L"]
    vs_base = value / PAPER_C3_1NODE_PAIRS_S if (full_c3 and not lags and not conv) else None

    if rank == 0:
        hist = np.bincount(E_host, minlength=E_max + 1)[1:].tolist()
        out = {
            "metric": (f"time-delay CCM (pair, lag) cross maps/sec, lags {lags[0]}..{lags[1]}" if lags else
                       f"CCM convergence test (pair, library size, sample) cross maps/sec, sizes {conv[0]}, "
                       f"{args.samples} samples" if conv else METRIC),
            "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": vs_base, "vs_baseline_ref": PAPER_C3_REF if vs_base else None,
            "dtype": "f32 kNN certified against f64 keys / " + ("u16-code lookup (EDM_LOOKUP_U16, fp32 arithmetic)"
                                                                   if args.lookup == "u16" else "f32 lookup"),
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {N} series x L={L}, E=1..{E_max}, tau={tau}, Tp={Tp}, "
                                   f"mode={args.mode}, exclude_self" + (", lookup=u16" if args.lookup == "u16" else ""),
                       "N": N, "L": L, "lookup": args.lookup,
                       "parallelism": f"library rows / series sharded over {world} GPU(s)",
                       "l2": "inputs larger than L2 (dataset %.0f MB, tables+tiles stream through L2)" % (N * L * 4 / 1e6)},
            "phase_ms_per_step": {"simplex": phases[0] / args.steps, "allgather_E": phases[1] / args.steps,
                                  "ccm": phases[2] / args.steps, "gather_rho": phases[3] / args.steps},
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
            "per_rank_ms_per_step": per_rank if world > 1 else None,
            "E_hist": hist, "k_bar": float((E_host + 1).mean()),
            "roofline": roofline_main, other_key: roofline_other,
            "cpu_baseline": cpu, "cpu_fast": cpu_fast, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
        }
        print(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
