OUT=gpurun_out
timeout 900 python bench.py --config c5 --N 1000 --L 40000 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/s2_L40k.log 2>&1
timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/s2_c5.log 2>&1
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $OUT/s2_c2.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/s2_c3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
echo done
