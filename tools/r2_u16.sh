#!/bin/bash
# 16-bit lookup: its tests, the fp32 parity tests (restructured lookup kernel), fp32 vs u16 bench lines
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lookup_u16.py -x -q -s > gpurun_out/u16_tests.log 2>&1
echo "u16 tests rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -x -q > gpurun_out/u16_parity.log 2>&1
echo "parity rc=$?"
for lk in fp32 u16 fp32 u16; do
  timeout 600 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --lookup $lk > gpurun_out/u16_bench_$lk.log 2>&1
  tail -1 gpurun_out/u16_bench_$lk.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lk', d['ms_per_step'], d['kernel_ms_per_step'])"
done
