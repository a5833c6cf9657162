#!/bin/bash
# One GPU call: the default bench line, the ncu launch list of a short bench command, and
# one ncu --set full capture each of the lookup and phase-2 kNN kernels at the bench config.
set -x
OUT=gpurun_out
timeout 900 python bench.py > $OUT/bench_default.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > $OUT/plain_short.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'lookup_kernel|knn_kernel<0' -s 600 -c 2 -o $OUT/prof_full $CMD > $OUT/ncu_full.log 2>&1
echo done
