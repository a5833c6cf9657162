#!/bin/bash
# ncu --set full captures of the phase-2 kNN and the lookup kernel at the bench config
# (run after the same command has exited 0 without ncu: tools/profile_round.sh)
OUT=gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > $OUT/plain_short.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lookup_kernel -s 100 -c 1 -o $OUT/prof_lookup $CMD > $OUT/ncu_lookup.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:knn_kernel -s 126 -c 1 -o $OUT/prof_knn $CMD > $OUT/ncu_knn.log 2>&1
echo done
