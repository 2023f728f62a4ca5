#!/bin/bash
set -x
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build.log 2>&1
python -c "import oracle; oracle.build()"
timeout 300 python tools/dbg_small.py > gpurun_out/dbg_small.log 2>&1; echo "dbg rc=$?" >> gpurun_out/dbg_small.log
EMU_TF32_A_LAYOUT=mn32 timeout 300 python tools/dbg_small.py > gpurun_out/dbg_small_mn32.log 2>&1; echo "dbg rc=$?" >> gpurun_out/dbg_small_mn32.log
timeout 300 python -m pytest tests/test_gpu_probe.py -q -s > gpurun_out/probe.log 2>&1; echo "rc=$?" >> gpurun_out/probe.log
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_split.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for mode in fp16 tf32; do
  timeout 300 python bench.py --steps 200 --warmup 10 --mode $mode --no-cpu-baseline > gpurun_out/bench_c2_$mode.log 2>&1
  timeout 300 python bench.py --steps 5 --warmup 3 --mode $mode --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_$mode.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches_c2_fp16.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm_kernel -s 3 -c 1 -o gpurun_out/prof_c2_fp16 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1
echo done
