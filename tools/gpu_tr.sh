#!/bin/bash
# trace + short A/B: bash tools/gpu_tr.sh TAG
TAG=${1:-tr}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
timeout 120 python tools/dbg_small.py > gpurun_out/dbg_$TAG.log 2>&1; RC=$?; echo "dbg rc=$RC" >> gpurun_out/dbg_$TAG.log
if [ $RC -ne 0 ]; then echo "dbg failed rc=$RC"; exit 1; fi
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/pytest_gemm_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_$TAG.log
timeout 300 python tools/trace.py fp16 > gpurun_out/trace_fp16_$TAG.log 2>&1
for r in 1 2 3; do for mode in fp16 tf32; do
  timeout 300 python bench.py --steps 300 --warmup 20 --mode $mode --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_${mode}_r${r}_$TAG.log 2>&1
done; done
timeout 300 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_fp16_$TAG.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --config c3 --mode tf32 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_tf32_$TAG.log 2>&1
