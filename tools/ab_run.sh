# A/B of library variants (VARIANTS env: base or lib suffixes) at c3 and c5 (short runs), then GPU tests
OUT=gpurun_out
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then unset LIBCCM_PATH; else export LIBCCM_PATH=$PWD/paper_2011_11082_b200/lib/libccm_$v.so; fi
  timeout 600 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/ab_c3_$v.log 2>&1
  timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/ab_c5_$v.log 2>&1
done
unset LIBCCM_PATH
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
echo done
