#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for mode in fp16 tf32; do for kb in 32 64 128 256 4096; do for mk in "512 1024" "1024 512" "256 256"; do
  timeout 20 python tools/kb_probe.py $mode $kb $mk >> gpurun_out/kbprobe.log 2>&1 || echo "FAIL $mode $kb $mk rc=$?" >> gpurun_out/kbprobe.log
done; done; done
cat gpurun_out/kbprobe.log
