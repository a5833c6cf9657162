#!/bin/bash
# One GPU call refreshing every round artefact: default bench line, launch list of a short
# bench command, and ncu --set full captures of the lookup and phase-2 kNN kernels.
OUT=gpurun_out
timeout 900 python bench.py > $OUT/bench_default.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > $OUT/plain_short.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lookup_kernel -s 100 -c 1 -o $OUT/prof_lookup $CMD > $OUT/ncu_lookup.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:knn_kernel -s 126 -c 1 -o $OUT/prof_knn $CMD > $OUT/ncu_knn.log 2>&1
echo done
