#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ "${NG:-1}" = "1" ]; then
  timeout 1800 python bench.py --config c4 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c4_1gpu.log 2>&1
else
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29619"
  timeout 1800 $TR bench.py --gpus $NG --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_${NG}gpu.log 2>&1
fi
echo done
