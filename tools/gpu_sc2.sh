#!/bin/bash
TAG=${1:-sc2}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_gemm.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
for V in "EMU_TS_SPLITC=1" "EMU_TS_SPLITC=1 EMU_TS_N=128" "EMU_TS_SPLITC=0"; do
  for mode in fp16 tf32; do
    env $V timeout 300 python bench.py --steps 300 --warmup 10 --mode $mode --no-cpu-baseline --no-e2e > "gpurun_out/bench_c2_${mode}_${V// /_}_$TAG.log" 2>&1
    env $V timeout 300 python bench.py --steps 5 --warmup 3 --mode $mode --config c3 --no-cpu-baseline --no-e2e > "gpurun_out/bench_c3_${mode}_${V// /_}_$TAG.log" 2>&1
  done
done
timeout 300 python tools/prof_roles.py c2 fp16 5 >> gpurun_out/prof_roles_$TAG.log 2>&1
timeout 300 python tools/prof_roles.py c3 fp16 3 >> gpurun_out/prof_roles_$TAG.log 2>&1
EMU_TS_N=128 timeout 300 python tools/prof_roles.py c3 tf32 3 >> gpurun_out/prof_roles_$TAG.log 2>&1
