set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" > gpurun_out/lscpu.txt
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/r2_plain_short.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_kernel -s 6 -c 1 -o gpurun_out/r2_knn_ccm $CMD > gpurun_out/r2_ncu_knn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_kernel -s 1 -c 1 -o gpurun_out/r2_knn_simplex $CMD > gpurun_out/r2_ncu_knn1.log 2>&1
echo done
