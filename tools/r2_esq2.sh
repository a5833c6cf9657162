#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/esq_stats.py > gpurun_out/esq_stats.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tables.py -x -q > gpurun_out/esq_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/esq_pytest.log
timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/esq_bench.log 2>&1
echo done
