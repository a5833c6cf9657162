#!/bin/bash
# GPU check: tests, smoke, short bench line; optional ncu source capture of the phase-2 kNN
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1
if [ -n "$NCU_KNN" ]; then
  CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_kernel -s 60 -c 1 -o gpurun_out/r2_knn_ccm $CMD > gpurun_out/r2_ncu_knn.log 2>&1
fi
echo done
