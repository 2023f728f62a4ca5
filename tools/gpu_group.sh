#!/bin/bash
# c3 raster-group sweep: bench + DRAM bytes per launch
TAG=${1:-grp}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > /dev/null 2>&1
for G in ${GS:-2 4 8 16 64}; do
  EMU_GROUP_M=$G timeout 300 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_fp16_g${G}_$TAG.log 2>&1
done
for G in ${GS:-2 4 8 16 64}; do
  EMU_GROUP_M=$G timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:emu_sgemm -s 3 -c 1 --csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3_g${G}_$TAG.csv 2>&1
done
