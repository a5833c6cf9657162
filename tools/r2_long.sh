#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_tables.py tests/test_gpu_long.py tests/test_gpu_parity.py -x -q -k "long or c5 or gmem or identical" > gpurun_out/long_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/long_pytest.log
timeout 1800 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --config c5 > gpurun_out/bench_c5.log 2>&1
echo done
