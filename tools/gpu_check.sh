#!/bin/bash
# quick state check: build, GPU tests, smoke, benches (no ncu).  bash tools/gpu_check.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1
timeout 600 python bench.py --mode tf32 > gpurun_out/bench_default_tf32_$TAG.log 2>&1
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/bench_c3_fp16_$TAG.log 2>&1
timeout 600 python bench.py --config c3 --mode tf32 --steps 20 --warmup 3 > gpurun_out/bench_c3_tf32_$TAG.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_$TAG.log gpurun_out/smoke_$TAG.log
for f in gpurun_out/bench_*_$TAG.log; do echo $f; tail -c 600 $f; echo; done
