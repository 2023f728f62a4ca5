#!/bin/bash
# first GPU contact: build, sanity, tests, bench, ncu (each step bounded)
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python paper_2308_15152_b200/build.py --force > gpurun_out/build.log 2>&1
python -c "import oracle; oracle.build(force=True)"
timeout 300 python tools/dbg_small.py > gpurun_out/dbg_small.log 2>&1; echo "dbg rc=$?" >> gpurun_out/dbg_small.log
timeout 300 python -m pytest tests/test_gpu_probe.py -x -q -s > gpurun_out/probe.log 2>&1; echo "rc=$?" >> gpurun_out/probe.log
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_split.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python -m pytest tests/test_gpu_split.py -q -x > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
tail -5 gpurun_out/*.log
