#!/usr/bin/env python
"""Oracle phase 1 (optimal E, Alg. 1 lines 2-10) over EVERY series of a
BASELINE config, written to tests/golden/<config>_optE_oracle.npz.

Calls only oracle/ (and the seeded generator synth.py): the stored optE is the oracle's, never
the CUDA path's. Used by tests/test_gpu_full_optE.py (full-N bit-exact optE parity) and by
bench.py --impl reference (the oracle's own E distribution for its phase-2 sample).

  python tools/oracle_full_optE.py --config c3 [--threads N]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2011_11082_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--chunk", type=int, default=4096)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    data = synth.make_config(a.config)
    L, N = data.shape
    t0 = time.time()
    optE = np.zeros(N, np.int8)
    for c0 in range(0, N, a.chunk):
        c1 = min(N, c0 + a.chunk)
        e, _ = O.simplex_all(data, cfg["E_max"], cfg["tau"], c0, c1, nthreads=a.threads)
        optE[c0:c1] = e
        print(f"{c1}/{N} series, {time.time() - t0:.0f} s", flush=True)
    out = os.path.join(ROOT, "tests", "golden", f"{a.config}_optE_oracle.npz")
    np.savez_compressed(out, optE=optE, config=a.config, N=N, L=L, E_max=cfg["E_max"], tau=cfg["tau"],
                        seed=synth.SEED_BASE + int(a.config[1:]), seconds=time.time() - t0, threads=a.threads,
                        source="oracle/ccm_oracle.c oracle_simplex_all (fp64), tools/oracle_full_optE.py")
    print("wrote", out, "hist", np.bincount(optE, minlength=21)[1:].tolist())


if __name__ == "__main__":
    main()
