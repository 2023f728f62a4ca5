#!/bin/bash
# build + sanity + benches (+ optional ncu): bash tools/gpu_perf.sh [tag] [ncu]
TAG=${1:-run}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1
python -c "import oracle; oracle.build()"
timeout 300 python tools/dbg_small.py > gpurun_out/dbg_$TAG.log 2>&1; echo "dbg rc=$?" >> gpurun_out/dbg_$TAG.log
for mode in fp16 tf32; do
  timeout 300 python bench.py --steps 200 --warmup 10 --mode $mode --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_${mode}_$TAG.log 2>&1
  timeout 300 python bench.py --steps 5 --warmup 3 --mode $mode --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_${mode}_$TAG.log 2>&1
done
if [ "$2" == "ncu" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm_kernel -s 3 -c 1 -o gpurun_out/prof_c2_fp16_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm_kernel -s 3 -c 1 -o gpurun_out/prof_c3_fp16_$TAG python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3_$TAG.log 2>&1
fi
echo done
