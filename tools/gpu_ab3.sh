#!/bin/bash
# robust A/B on c2: each env variant benched REPS times, interleaved (1000 steps each)
TAG=$1; shift
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
[ -n "$TESTENV" ] && { env $TESTENV timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "astat or c2_full" > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log; }
for r in $(seq ${REPS:-3}); do
  for mode in ${MODES:-fp16 tf32}; do
    i=0; for V in "$@"; do
      env $V timeout 300 python bench.py --steps ${STEPS:-300} --warmup 20 --mode $mode --no-cpu-baseline --no-e2e > "gpurun_out/bench_c2_${mode}_v${i}_r${r}_$TAG.log" 2>&1; i=$((i+1))
    done
  done
done
