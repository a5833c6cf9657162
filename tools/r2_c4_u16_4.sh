#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29639"
timeout 1800 $TR bench.py --gpus 4 --config c4 --steps 3 --warmup 3 --lookup u16 > gpurun_out/bench_c4_u16_4gpu.log 2>&1
echo done
