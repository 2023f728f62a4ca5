#!/bin/bash
TAG=${1:-tt}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_trans.py -q -x > gpurun_out/pytest_trans_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_trans_$TAG.log
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_range.py -q -x > gpurun_out/pytest_gemm_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_$TAG.log
for mode in fp16 tf32; do
  timeout 300 python bench.py --steps 300 --warmup 20 --mode $mode --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_${mode}_$TAG.log 2>&1
done
