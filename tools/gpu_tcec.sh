#!/bin/bash
# device-API check: build, tcec GPU tests, timings.  bash tools/gpu_tcec.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tcec.py -q -x -rf > gpurun_out/pytest_tcec_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tcec_$TAG.log
tail -n 30 gpurun_out/pytest_tcec_$TAG.log
timeout 300 python tools/tcec_time.py > gpurun_out/tcec_time_$TAG.log 2>&1
tail -n 5 gpurun_out/tcec_time_$TAG.log
