OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
timeout 600 python bench.py --config c2 --convergence 25,50,100,200,400,999 --samples 4 > $OUT/bench_conv_c2.log 2>&1
timeout 900 python bench.py --config c3 --N 8192 --convergence 100,400,1449 --samples 2 > $OUT/bench_conv_c3_8k.log 2>&1
timeout 1200 python bench.py --config c5 --N 1000 --L 40000 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $OUT/bench_L40k.log 2>&1
echo done
