#!/bin/bash
# parity (tables + parity) then short bench lines per env variant
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tables.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
for v in ${VARIANTS:-default}; do
  if [ "$v" = "default" ]; then env=""; else env="$v"; fi
  env $env timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab_bench_$(echo $v | tr "=,/." "____").log 2>&1
done
echo done
