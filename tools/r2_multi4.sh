#!/bin/bash
# 4-GPU: byte-identical c3 map vs one GPU; c3 and c4 bench lines
cd "${GRAFT_REPO_ROOT:-.}"
NG=4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29613"
timeout 2400 $TR tools/multi_identical.py --config c3 > gpurun_out/multi_identical_c3_4gpu.log 2>&1
timeout 1500 $TR bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_c3_4gpu.log 2>&1
timeout 2400 $TR bench.py --gpus 4 --steps 3 --warmup 3 --config c4 > gpurun_out/bench_c4_4gpu.log 2>&1
echo done
