#!/bin/bash
# 16-bit lookup at NG GPUs: c3 bench line and the byte-identity check of the distributed map
cd "${GRAFT_REPO_ROOT:-.}"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29627"
timeout 1500 $TR bench.py --gpus $NG --steps 3 --warmup 3 --lookup u16 > gpurun_out/bench_c3_u16_${NG}gpu.log 2>&1
timeout 2400 $TR tools/multi_identical.py --config c3 --lookup u16 > gpurun_out/multi_identical_c3_u16_${NG}gpu.log 2>&1
echo done
