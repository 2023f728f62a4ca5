#!/bin/bash
# interleaved timing of several prebuilt libraries (abtmp/*): bash tools/gpu_bisect.sh TAG LIB...
TAG=$1; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/bisect_$TAG.smi
timeout 1200 python tools/ab_lib.py "$@" > gpurun_out/bisect_$TAG.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/bisect_$TAG.json')); print(json.dumps(d['libs'])); print(json.dumps(d['mean']))"
