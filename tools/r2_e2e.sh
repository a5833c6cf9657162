#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py -q -k "host or abi or export" > gpurun_out/e2e_pytest.log 2>&1; echo rc=$? >> gpurun_out/e2e_pytest.log
timeout 1200 python bench.py --steps 1 --warmup 1 --e2e-steps 5 --no-cpu-baseline > gpurun_out/bench_e2e.log 2>&1
echo done
