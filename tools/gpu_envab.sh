#!/bin/bash
# A/B of env-selected kernel variants.
#   TESTENV="EMU_X=1" bash tools/gpu_envab.sh TAG "EMU_X=0" "EMU_X=1" ...
# parity tests (test_gpu_gemm.py) run under $TESTENV; every variant is benched on
# c2/c3 x fp16/tf32 (variants interleaved per workload) and role-timed on c2/c3 fp16.
TAG=$1; shift
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
env $TESTENV timeout 120 python tools/dbg_small.py > gpurun_out/dbg_$TAG.log 2>&1; RC=$?; echo "dbg rc=$RC" >> gpurun_out/dbg_$TAG.log
if [ $RC -ne 0 ]; then echo "dbg failed rc=$RC"; exit 1; fi
env $TESTENV timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/pytest_gemm_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_$TAG.log
for mode in fp16 tf32; do
  i=0; for V in "$@"; do
    env $V timeout 300 python bench.py --steps 300 --warmup 10 --mode $mode --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_${mode}_v${i}_$TAG.log 2>&1; i=$((i+1))
  done
  i=0; for V in "$@"; do
    env $V timeout 300 python bench.py --steps 5 --warmup 3 --mode $mode --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_${mode}_v${i}_$TAG.log 2>&1; i=$((i+1))
  done
done
i=0; for V in "$@"; do
  echo "== v$i: $V" >> gpurun_out/prof_roles_$TAG.log
  env $V timeout 300 python tools/prof_roles.py c2 fp16 5 >> gpurun_out/prof_roles_$TAG.log 2>&1
  env $V timeout 300 python tools/prof_roles.py c3 fp16 3 >> gpurun_out/prof_roles_$TAG.log 2>&1
  i=$((i+1))
done
