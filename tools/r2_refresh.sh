#!/bin/bash
# Round-2 GPU refresh: all GPU tests, smoke, the default bench line, the launch list of a short
# bench command and ncu --set full captures of the lookup and the phase-2 kNN (E-sequential).
cd "${GRAFT_REPO_ROOT:-.}"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench_default.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lookup_kernel -s 100 -c 1 -o $OUT/prof_lookup $CMD > $OUT/ncu_lookup.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:knn_eseq -s 60 -c 1 -o $OUT/prof_knn $CMD > $OUT/ncu_knn.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:knn_eseq -s 2 -c 1 -o $OUT/prof_knn1 $CMD > $OUT/ncu_knn1.log 2>&1
echo done
