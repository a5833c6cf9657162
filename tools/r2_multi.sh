#!/bin/bash
# 2/4-GPU: byte-identical maps vs one GPU, and the bench lines (target mode; library mode dealing)
cd "${GRAFT_REPO_ROOT:-.}"
NG=${NG:-2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29611"
timeout 1500 $TR tools/multi_identical.py --config c2 > gpurun_out/multi_identical_c2_${NG}gpu.log 2>&1
timeout 2400 $TR tools/multi_identical.py --config c3 > gpurun_out/multi_identical_c3_${NG}gpu.log 2>&1
timeout 1500 $TR bench.py --gpus $NG --steps 3 --warmup 3 > gpurun_out/bench_c3_${NG}gpu.log 2>&1
timeout 1500 $TR bench.py --gpus $NG --steps 3 --warmup 3 --mode library --e2e-steps 0 > gpurun_out/bench_c3_library_${NG}gpu.log 2>&1
echo done
