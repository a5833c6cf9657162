"""GPU vs fast-CPU time of the whole causal map (phase 1 + phase 2) at N = 1,000 series and a
growing number of time steps -- the paper's GPU-speedup experiment ("GPU speedup with
varying number of time steps (1,000 time series)"). GPU: one B200, CUDA events around both
phases (inputs resident). CPU: cpu_baseline/ (the fast host implementation, bit-identical to the
oracle) on the box's host cores, timed on a bounded sample and extrapolated (bench.oracle_sample).
Prints one JSON object; run on the GPU box:  python tools/speedup_vs_L.py > profiles/...json"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2011_11082_b200 import build, libccm, synth  # noqa: E402

Ls = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1000,2000,5000,10000,20000,40000").split(",")]
N = 1000
build.build()
libccm.load()
rows = []
for L in Ls:
    host = synth.make_config("c5", N=N, L=L)
    d = torch.from_numpy(host).cuda()
    st = torch.cuda.current_stream()
    for it in range(2):  # warm-up, then timed
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        E = libccm.simplex_optimal_E(d, 20)
        rho = libccm.ccm_all_pairs(d, E)
        e1.record(st)
        torch.cuda.synchronize()
    gpu_s = e0.elapsed_time(e1) / 1e3
    E_host = E.cpu().numpy()
    v, secs, cores, desc = bench.oracle_sample(host, E_host, "target", 1, 1, N, N, impl="fast", budget_s=15.0)
    cpu_s = N * N / v
    rows.append({"L": L, "N": N, "gpu_s": gpu_s, "cpu_fast_s": cpu_s, "speedup": cpu_s / gpu_s, "cpu_cores": cores,
                 "cpu_sample": desc})
    print(json.dumps(rows[-1]), file=sys.stderr)
    del d, rho
    libccm.release_workspaces()
    torch.cuda.empty_cache()
print(json.dumps({"experiment": "GPU (1 x B200) vs fast CPU, whole causal map, N=1000, E_max=20, tau=1, Tp=1",
                  "paper": "P:793-796: 1 GPU slower than CPU at L <= 2,000, faster from 5,000; 3.5x at 40,000 "
                           "(V100 vs one CPU socket)", "rows": rows}))
