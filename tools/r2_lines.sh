#!/bin/bash
# round-2 lines for the non-headline workloads (f1 lags, c5, library mode 1 GPU) + the new table test
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tables.py -q -k "identical or c3" > gpurun_out/lines_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lines_pytest.log
timeout 1200 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline "--lags=-2:2" > gpurun_out/bench_c3_lags.log 2>&1
timeout 1200 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --mode library > gpurun_out/bench_c3_library.log 2>&1
timeout 1800 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --config c5 > gpurun_out/bench_c5.log 2>&1
echo done
