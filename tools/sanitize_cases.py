#!/usr/bin/env python
"""Small invocations of every libccm kernel variant for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): phase 1 (E-sequential kNN, SIMPLEX), phase 2 target mode (E-sequential kNN +
smem lookup + TMA ring), library mode (sweep kNN with per-slot E), the padded-global-series kNN,
the convergence test (library-set mask), time-delay lags, edm_embed_knn, the long-series lookup
(global gathers), the table readback, quantised data (exact-tie fallback) and a constant series
(tie flood). Usage: compute-sanitizer --tool <tool> python tools/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_11082_b200 import libccm, synth  # noqa: E402

libccm.load()
dev = lambda a, dt=torch.float32: torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dt)

d1 = synth.make_config("c1")
data = synth.random_dataset(40, 160, 3)
data[:, 7] = 0.5                      # constant series: tie flood
data = np.concatenate([data, synth.quantise8(synth.make_config("c2", N=8, L=160))], axis=1)  # exact ties
d = dev(data)
E = libccm.simplex_optimal_E(d, 8)
Eh = E.cpu().numpy()
libccm.simplex_optimal_E(dev(d1), 10)
libccm.ccm_all_pairs(d, E, 1, 1, "target")
libccm.ccm_all_pairs(d, E, 1, 0, "library")
libccm.ccm_rows(d, E, np.array([5, 1, 7, 30], np.int32), 1, 1, "library")
libccm.ccm_lagged(d, E, 1, -2, 2, "target")
libccm.ccm_convergence(d, E, [12, 40, 159], synth.library_orders(2, 160, 1), 1, 1, "target", samples=True)
libccm.ccm_tables(d, E, int(Eh[0]), 1, 1)
libccm.embed_knn(d[:, 3].contiguous(), 3, 1, 1, True)
os.environ["CCM_KNN_SERIES"] = "global"
libccm.simplex_optimal_E(d, 8, 2)
libccm.ccm_all_pairs(d, E, 2, 1, "target")
del os.environ["CCM_KNN_SERIES"]
os.environ["CCM_KNN_ALGO"] = "sweep"
libccm.simplex_optimal_E(d, 8)
libccm.ccm_all_pairs(d, E, 1, 1, "target")
del os.environ["CCM_KNN_ALGO"]
# 16-bit lookup targets: the code path, and a flagged 64-tile (heavy tail) on the fp32 fallback
libccm.ccm_all_pairs(d, E, 1, 1, "target", lookup="u16")
libccm.ccm_all_pairs(d, E, 1, 0, "library", lookup="u16")
libccm.ccm_lagged(d, E, 1, -2, 2, "target", lookup="u16")
ht = synth.make_config("c2", N=150, L=200)
ht[50, 100] += 1e3
dh = dev(ht)
libccm.ccm_all_pairs(dh, libccm.simplex_optimal_E(dh, 6), 1, 1, "library", lookup="u16")
long = dev(synth.make_config("c5", N=12, L=2100))  # target tiles beyond shared memory: global gathers
libccm.ccm_all_pairs(long, dev(np.arange(1, 13) % 6 + 1, torch.int32), 1, 1, "target", True, 0, 3)
torch.cuda.synchronize()
print("sanitize cases done")
