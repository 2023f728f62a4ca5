#!/bin/bash
# rebuild, targeted GPU tests, interleaved timing vs prebuilt libraries.  bash tools/gpu_fix.sh TAG LIB...
TAG=$1; shift
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 1200 python tools/ab_lib.py "$@" paper_2308_15152_b200/libemusgemm.so 2 > gpurun_out/ab_$TAG.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/ab_$TAG.json')); print(json.dumps(d['libs'])); print(json.dumps(d['mean']))"
