#!/bin/bash
# ncu captures of the current kernel: bash tools/gpu_ncu.sh TAG
TAG=${1:-n}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c2_fp16_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c2_tf32_$TAG python bench.py --mode tf32 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2t_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c3_fp16_$TAG python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 20 --csv --log-file gpurun_out/launches_c2_fp16_$TAG.csv python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
