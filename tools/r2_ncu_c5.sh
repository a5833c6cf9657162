#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --config c5 --N 2048"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:knn_long -s 3 -c 1 -o gpurun_out/r2_c5_knn $CMD > gpurun_out/r2_ncu_c5.log 2>&1
echo done
