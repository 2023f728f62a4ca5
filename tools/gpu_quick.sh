#!/bin/bash
# quick check: build, TC accumulation samples, GPU tests.  bash tools/gpu_quick.sh TAG
TAG=${1:-q}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_$TAG.log; exit 1; }
python -c "import oracle; oracle.build()"
timeout 600 python tools/tc_collect.py > gpurun_out/tc_collect_$TAG.log 2>&1; echo "tc rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
