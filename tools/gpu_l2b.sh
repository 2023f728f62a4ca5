#!/bin/bash
# repeated, interleaved L2-hint comparison on c3 (fp16/tf32) and c2.  bash tools/gpu_l2b.sh TAG
TAG=$1
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
for rep in 1 2 3; do for P in 0 1 3; do for MODE in fp16 tf32; do
  r=$(EMU_L2_POLICY=$P timeout 300 python bench.py --config c3 --mode $MODE --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'])")
  echo "rep=$rep pol=$P c3_$MODE $r" | tee -a gpurun_out/l2_$TAG.txt
done; done; done
for rep in 1 2; do for P in 0 1; do
  r=$(EMU_L2_POLICY=$P timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'])")
  echo "rep=$rep pol=$P c2_fp16 $r" | tee -a gpurun_out/l2_$TAG.txt
done; done
