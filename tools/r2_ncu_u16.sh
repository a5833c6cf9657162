#!/bin/bash
# ncu --set full of one c3 lookup launch with the 16-bit lookup targets
cd "${GRAFT_REPO_ROOT:-.}"
OUT=gpurun_out/u16ncu; mkdir -p $OUT
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --lookup u16"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lookup_kernel -s 100 -c 1 -o $OUT/prof_lookup_u16 $CMD > $OUT/ncu_lookup.log 2>&1
echo rc=$?
