#!/bin/bash
python paper_2308_15152_b200/build.py > /dev/null 2>&1
rm -f gpurun_out/prof_roles_c2ts.log
for md in fp16 tf32; do EMU_KERNEL=ts timeout 300 python tools/prof_roles.py c2 $md 5 >> gpurun_out/prof_roles_c2ts.log 2>&1; done
EMU_KERNEL=ts timeout 300 python tools/prof_roles.py c3 fp16 3 >> gpurun_out/prof_roles_c2ts.log 2>&1
