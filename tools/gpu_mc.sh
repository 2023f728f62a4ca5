#!/bin/bash
# multicast / sharded checks + tcec tests.  bash tools/gpu_mc.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multicast.py tests/test_gpu_tcec.py -q -rf > gpurun_out/pytest_mc_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mc_$TAG.log
tail -n 30 gpurun_out/pytest_mc_$TAG.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/bench_c3_sharded1_$TAG.log 2>&1
tail -c 1500 gpurun_out/bench_c3_sharded1_$TAG.log
