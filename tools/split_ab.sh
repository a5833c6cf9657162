OUT=gpurun_out
for v in 0 148; do
  CCM_LK_SPLIT=$v timeout 600 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/split_c3_$v.log 2>&1
  CCM_LK_SPLIT=$v timeout 600 python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/split_c4_$v.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
echo done
