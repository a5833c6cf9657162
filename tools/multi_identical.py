#!/usr/bin/env python
"""Byte-identity of the causal map across world sizes on real GPUs:
under torchrun, every rank computes its share (target mode: contiguous row blocks; library mode:
rows dealt over the E-sorted order) through distributed.causal_map_distributed and gathers to rank
0, which also computes the whole map alone on its own GPU and compares the two bit for bit.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/multi_identical.py --config c3
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_11082_b200 import distributed, libccm, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--N", type=int, default=None)
ap.add_argument("--lookup", default="fp32", choices=["fp32", "u16"])
a = ap.parse_args()
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, world = dist.get_rank(), dist.get_world_size()
libccm.load()
data = torch.from_numpy(synth.make_config(a.config, N=a.N)).to(dev)
L, N = data.shape
out = {"config": a.config, "N": N, "L": L, "world": world, "lookup": a.lookup}
for mode in ("target", "library"):
    t0 = time.time()
    E, rows, full = distributed.causal_map_distributed(data, 20, 1, 1, mode, True, lookup=a.lookup)
    torch.cuda.synchronize()
    out[f"{mode}_distributed_s"] = time.time() - t0
    if rank == 0:
        E1, rho1 = libccm.causal_map(data, 20, 1, 1, mode, True, lookup=a.lookup)
        torch.cuda.synchronize()
        out[f"{mode}_optE_identical"] = bool(torch.equal(E.cpu(), E1.cpu()))
        out[f"{mode}_map_identical"] = bool(torch.equal(full.view(torch.int32), rho1.view(torch.int32)))
        out[f"{mode}_nan_count"] = int(torch.isnan(rho1).sum())
        del rho1, full
    dist.barrier()
    torch.cuda.empty_cache()
if rank == 0:
    print(json.dumps(out))
dist.destroy_process_group()
