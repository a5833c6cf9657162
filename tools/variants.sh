for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then unset LIBCCM_PATH; else export LIBCCM_PATH=$PWD/paper_2011_11082_b200/lib/libccm_$v.so; fi
  timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/var_$v.log 2>&1
done
echo done
