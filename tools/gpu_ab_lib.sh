#!/bin/bash
# A/B: the in-tree library vs abtmp/old (another commit's build), plus KB sweeps.  bash tools/gpu_ab_lib.sh TAG
TAG=${1:-abl}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python tools/ab_lib.py abtmp/old/paper_2308_15152_b200/libemusgemm.so paper_2308_15152_b200/libemusgemm.so 3 > gpurun_out/ab_$TAG.json 2>&1
timeout 300 python tools/kb_c2.py > gpurun_out/kbc2_$TAG.json 2>&1
timeout 600 python tools/kb_sweep.py 16384 > gpurun_out/kbc3_$TAG.json 2>&1
cat gpurun_out/ab_$TAG.json gpurun_out/kbc2_$TAG.json; head -3 gpurun_out/kbc3_$TAG.json
