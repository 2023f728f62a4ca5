#!/bin/bash
# c2 tf32 under the selectable kernel configurations.  bash tools/gpu_tf32cfg.sh TAG
TAG=$1
mkdir -p gpurun_out
run() { r=$(env "$@" timeout 300 python bench.py --mode tf32 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'])"); echo "$* -> $r" | tee -a gpurun_out/tf32cfg_$TAG.txt; }
for rep in 1 2; do
  run X=default
  run EMU_TS_N=96
  run EMU_TS_SPLITC=0
  run EMU_KERNEL=pair
  run EMU_L2_POLICY=0
done
