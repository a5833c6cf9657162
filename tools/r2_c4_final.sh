#!/bin/bash
# c4 on one GPU, W=3 K=3: the fp32 headline kernels and the 16-bit lookup option
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1800 python bench.py --config c4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c4_1gpu.log 2>&1
timeout 1800 python bench.py --config c4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --lookup u16 > gpurun_out/bench_c4_u16_1gpu.log 2>&1
echo done
