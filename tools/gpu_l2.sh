#!/bin/bash
# c3 raster group x L2 hint sweep (TS kernel).  bash tools/gpu_l2.sh TAG
TAG=$1
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
for G in 2 4; do for P in 0 1 2 3; do
  r=$(EMU_GROUP_M=$G EMU_L2_POLICY=$P timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'])")
  echo "group=$G pol=$P c3_fp16 $r" | tee -a gpurun_out/l2_$TAG.txt
done; done
