OUT=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
timeout 900 python bench.py > $OUT/bench_default.log 2>&1
timeout 1800 python tools/speedup_vs_L.py > $OUT/speedup_vs_L.json 2> $OUT/speedup_vs_L.err
lscpu > $OUT/lscpu.txt 2>&1
echo done
