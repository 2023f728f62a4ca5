#!/bin/bash
python paper_2308_15152_b200/build.py > /dev/null 2>&1
cat > /tmp/c3l2.py <<'PY'
import torch, sys, os, json
sys.path.insert(0, os.getcwd())
import paper_2308_15152_b200 as emu
m = n = k = 16384
A = torch.rand(k, m, device="cuda") * 2 - 1
B = torch.rand(n, k, device="cuda") * 2 - 1
C = torch.empty(n, m, device="cuda")
for _ in range(2):
    emu.emu_sgemm(m, n, k, 1.0, A, m, B, k, 0.0, C, m, "fp16")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    emu.emu_sgemm(m, n, k, 1.0, A, m, B, k, 0.0, C, m, "fp16")
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(json.dumps({"gm": os.environ.get("EMU_GROUP_M"), "pol": os.environ.get("EMU_L2_POLICY"), "ms": ms, "tf": 2 * m**3 / ms / 1e9}))
PY
for gm in 16 4 8 32; do for pol in 0 1 3; do
  EMU_GROUP_M=$gm EMU_L2_POLICY=$pol timeout 120 python /tmp/c3l2.py >> gpurun_out/c3_l2.log 2>&1
done; done
EMU_GROUP_M=8 EMU_L2_POLICY=1 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:emu_sgemm -s 2 -c 1 python /tmp/c3l2.py > gpurun_out/c3_l2_ncu.log 2>&1
EMU_GROUP_M=16 EMU_L2_POLICY=0 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:emu_sgemm -s 2 -c 1 python /tmp/c3l2.py >> gpurun_out/c3_l2_ncu.log 2>&1
