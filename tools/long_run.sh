OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
timeout 1500 python bench.py --config c5 --N 1000 --L 40000 --e2e-steps 1 --cpu-sample 16 > $OUT/bench_L40k.log 2>&1
CCM_KNN_SERIES=smem timeout 900 python bench.py --config c5 --N 1000 --L 40000 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/bench_L40k_smem.log 2>&1
timeout 1500 python bench.py --config c5 --e2e-steps 1 --cpu-sample 16 > $OUT/bench_c5.log 2>&1
echo done
