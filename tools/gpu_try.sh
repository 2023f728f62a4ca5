#!/bin/bash
# quick kernel experiment: targeted GPU tests + interleaved timing vs prebuilt libraries + a c2 bench line.
#   bash tools/gpu_try.sh TAG LIB...
TAG=$1; shift
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_bitexact.py tests/test_gpu_gemm.py -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 1200 python tools/ab_lib.py "$@" paper_2308_15152_b200/libemusgemm.so 2 > gpurun_out/ab_$TAG.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/ab_$TAG.json')); print(json.dumps(d['libs'])); print(json.dumps(d['mean']))"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.log | cut -c1-200

