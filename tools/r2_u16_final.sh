#!/bin/bash
# 16-bit lookup: full bench line (c3, 1 GPU, with e2e and cpu baseline) + ncu --set full of one lookup launch
cd "${GRAFT_REPO_ROOT:-.}"
OUT=gpurun_out/u16ncu; mkdir -p $OUT
timeout 900 python bench.py --lookup u16 > gpurun_out/u16_bench_full.log 2>&1
echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --lookup u16"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lookup_kernel -s 100 -c 1 -o $OUT/prof_lookup_u16 -f $CMD > $OUT/ncu_lookup.log 2>&1
echo "ncu rc=$?"
