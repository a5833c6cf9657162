#!/bin/bash
# interleaved env-variant short bench lines, each twice
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
for v in ${VARIANTS}; do
  env $v timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/envab_$(echo $v | tr "=,/." "____")_$rep.log 2>&1
done; done
echo done
