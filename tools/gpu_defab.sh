#!/bin/bash
# A/B of compile-time variants: bash tools/gpu_defab.sh TAG "-DX=1" "-DX=2" ...
# (EMU_BUILD_DEFS for build.py) each variant: build, c2 parity subset, c2 fp16/tf32 x3 and c3 fp16/tf32 benches
TAG=$1; shift
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
i=0
for D in "$@"; do
  EMU_BUILD_DEFS="$D" python paper_2308_15152_b200/build.py --force > gpurun_out/build_${TAG}_v$i.log 2>&1 || { echo "BUILD FAILED $D"; i=$((i+1)); continue; }
  timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "astat or c2_full or parity_uniform or identity" > gpurun_out/pytest_${TAG}_v$i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}_v$i.log
  for r in 1 2 3; do for mode in fp16 tf32; do
    timeout 300 python bench.py --steps 300 --warmup 20 --mode $mode --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_${mode}_v${i}_r${r}_$TAG.log 2>&1
  done; done
  for mode in fp16 tf32; do
    timeout 300 python bench.py --steps 10 --warmup 3 --config c3 --mode $mode --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_${mode}_v${i}_$TAG.log 2>&1
  done
  i=$((i+1))
done
python paper_2308_15152_b200/build.py --force > /dev/null 2>&1
