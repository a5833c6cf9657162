OUT=gpurun_out
timeout 1500 python bench.py --config c5 --e2e-steps 1 > $OUT/bench_c5.log 2>&1
timeout 1500 python bench.py --config c5 --N 1000 --L 40000 --e2e-steps 1 > $OUT/bench_L40k.log 2>&1
timeout 1200 python bench.py --lags=-2:2 > $OUT/bench_lags.log 2>&1
timeout 900 python bench.py --mode library --e2e-steps 3 > $OUT/bench_c3_library.log 2>&1
timeout 600 python bench.py --config c2 --convergence 25,50,100,200,400,999 --samples 4 > $OUT/bench_conv_c2.log 2>&1
echo done
