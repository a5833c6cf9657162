# 2 / 4-GPU bench lines (run with gpurun --gpus N; N from $NG)
OUT=gpurun_out
NG=${NG:-2}
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG > $OUT/bench_c3_${NG}gpu.log 2>&1
if [ "$NG" = "4" ]; then
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus $NG --config c5 --N 1000 --L 40000 > $OUT/bench_L40k_${NG}gpu.log 2>&1
fi
echo done
