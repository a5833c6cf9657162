#!/usr/bin/env python
"""Counters of the E-sequential kNN (debug build lib/libccm_stats.so, -DCCM_ESQ_STATS) on one c3
block: flagged candidates, rounds, seeds, fillers per (query, E)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["LIBCCM_PATH"] = os.path.join(ROOT, "paper_2011_11082_b200", "lib", "libccm_stats.so")
from paper_2011_11082_b200 import libccm, synth  # noqa: E402

lib = libccm.load()
lib.edm_debug_esq_stats.argtypes = [C.c_void_p]
data = synth.make_config("c3", N=int(os.environ.get("N", "4096")))
d = torch.from_numpy(data).cuda()
st = np.zeros((21, 8), np.uint64)
for name, fn in (("phase1", lambda: libccm.simplex_optimal_E(d, 20)),
                 ("phase2", lambda: libccm.ccm_all_pairs(d, torch.from_numpy((1 + np.arange(d.shape[1]) % 20).astype(np.int32)).cuda(), 1, 1, "target", True, 0, 256))):
    lib.edm_debug_esq_stats(st.ctypes.data)
    fn()
    torch.cuda.synchronize()
    lib.edm_debug_esq_stats(st.ctypes.data)
    cnt = st[:, 6].astype(float)
    print(name, "per (query, E): flagged / batches / carried seeds / S1 seeds / fillers / theta=inf / exact fallbacks")
    for E in range(1, 21):
        if cnt[E]:
            print(f"  E={E:2d} " + " ".join(f"{st[E, i] / cnt[E]:7.2f}" for i in (0, 1, 2, 3, 4, 5, 7)))
