#!/bin/bash
TAG=${1:-as}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
timeout 120 python tools/dbg_small.py > gpurun_out/dbg_$TAG.log 2>&1; RC=$?; echo "dbg rc=$RC" >> gpurun_out/dbg_$TAG.log
if [ $RC -ne 0 ]; then echo "dbg failed rc=$RC"; exit 1; fi
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "astat" > gpurun_out/pytest_astat_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_astat_$TAG.log
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/pytest_gemm_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_$TAG.log
for V in "EMU_TS_ASTAT=1" "EMU_TS_ASTAT=0"; do
  for mode in fp16 tf32; do
    env $V timeout 300 python bench.py --steps 300 --warmup 10 --mode $mode --no-cpu-baseline --no-e2e > "gpurun_out/bench_c2_${mode}_${V// /_}_$TAG.log" 2>&1
  done
done
timeout 300 python tools/prof_roles.py c2 fp16 5 >> gpurun_out/prof_roles_$TAG.log 2>&1
timeout 300 python tools/prof_roles.py c2 tf32 5 >> gpurun_out/prof_roles_$TAG.log 2>&1
