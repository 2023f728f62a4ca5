#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_kb2.log 2>&1 || { tail -20 gpurun_out/build_kb2.log; exit 1; }
rm -f gpurun_out/kbprobe2.log
for mode in fp16 tf32; do for kb in 128 160 192 256 4096; do for mk in "512 1024" "256 256"; do
  timeout 20 python tools/kb_probe.py $mode $kb $mk >> gpurun_out/kbprobe2.log 2>&1 || echo "FAIL $mode $kb $mk rc=$?" >> gpurun_out/kbprobe2.log
done; done; done
cat gpurun_out/kbprobe2.log
if grep -q FAIL gpurun_out/kbprobe2.log; then exit 1; fi
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -rf > gpurun_out/pytest_gemm_kb2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm_kb2.log
tail -5 gpurun_out/pytest_gemm_kb2.log
timeout 600 python tools/kb_sweep.py > gpurun_out/kb_sweep.json 2>&1
tail -2 gpurun_out/kb_sweep.json
