#!/bin/bash
# c3 raster group sweep with the default L2 hints.  bash tools/gpu_group2.sh TAG
TAG=$1
mkdir -p gpurun_out
for rep in 1 2; do for G in 2 3 1; do
  r=$(EMU_GROUP_M=$G timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'])")
  echo "rep=$rep group=$G c3_fp16 $r" | tee -a gpurun_out/group2_$TAG.txt
done; done
