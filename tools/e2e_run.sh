OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host or c1 or split" > $OUT/pytest_e2e.log 2>&1
timeout 900 python bench.py > $OUT/bench_default.log 2>&1
echo done
