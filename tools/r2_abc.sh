#!/bin/bash
# interleaved A/B/C short bench lines of prebuilt libraries (each twice)
cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do
for v in ${LIBS:-A D C}; do
  LIBCCM_PATH=paper_2011_11082_b200/lib/libccm_$v.so timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline $EXTRA > gpurun_out/abc_${v}_$rep.log 2>&1
done; done
echo done
