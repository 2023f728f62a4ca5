#!/bin/bash
python paper_2308_15152_b200/build.py > /dev/null 2>&1
rm -f gpurun_out/prof_roles_c2.log
for K in ts pair; do for md in fp16 tf32; do EMU_KERNEL=$K timeout 300 python tools/prof_roles.py c2 $md 5 >> gpurun_out/prof_roles_c2.log 2>&1; done; done
