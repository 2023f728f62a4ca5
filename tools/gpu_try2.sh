#!/bin/bash
# build, ALL GPU tests, c4 + c2 + c3 bench lines.  bash tools/gpu_try2.sh TAG
TAG=$1
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
tail -4 gpurun_out/pytest_$TAG.log
for c in c4 c2 c3; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$TAG.log 2>&1; tail -1 gpurun_out/bench_${c}_$TAG.log | cut -c1-160; done
