#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lookup_u16.py -x -q -s > gpurun_out/u16_tests.log 2>&1
echo "u16 tests rc=$?"
timeout 900 python bench.py --lookup u16 > gpurun_out/u16_bench_full.log 2>&1
echo "bench rc=$?"
