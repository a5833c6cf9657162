#!/bin/bash
# final-code multi-GPU lines: c3 bench (target) and the byte-identity check at NG GPUs
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29617"
timeout 1500 $TR bench.py --gpus $NG --steps 3 --warmup 3 > gpurun_out/bench_c3_${NG}gpu.log 2>&1
timeout 2400 $TR tools/multi_identical.py --config c3 > gpurun_out/multi_identical_c3_${NG}gpu.log 2>&1
echo done
