#!/bin/bash
python paper_2308_15152_b200/build.py > /dev/null 2>&1
cat > /tmp/c3small.py <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2308_15152_b200 as emu
m = n = k = 8192
A = torch.rand(k, m, device="cuda") * 2 - 1
B = torch.rand(n, k, device="cuda") * 2 - 1
C = torch.empty(n, m, device="cuda")
mode = sys.argv[1]
for _ in range(3):
    emu.emu_sgemm(m, n, k, 1.0, A, m, B, k, 0.0, C, m, mode)
torch.cuda.synchronize()
PY
for K in ts pair; do
EMU_KERNEL=$K timeout 600 ncu --set full --clock-control none -k regex:emu_sgemm -s 2 -c 1 -o gpurun_out/prof_c3s_fp16_$K python /tmp/c3small.py fp16 > gpurun_out/ncu_c3s_$K.log 2>&1
done
