#!/bin/bash
TAG=${1:-t}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1
python -c "import oracle; oracle.build()"
timeout 1500 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_split.py::test_split_bit_exact_all_inputs > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -m pytest tests/test_gpu_split.py -q > gpurun_out/pytest_split_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1
