#!/bin/bash
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > /dev/null 2>&1
rm -f gpurun_out/prof_roles.log
for c in c2 c3; do for md in fp16 tf32; do timeout 300 python tools/prof_roles.py $c $md 3 >> gpurun_out/prof_roles.log 2>&1; done; done

