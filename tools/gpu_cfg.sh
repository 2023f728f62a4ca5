#!/bin/bash
# layout tests + bench on every config.  bash tools/gpu_cfg.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_layout.py -q -rf > gpurun_out/pytest_layout_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_layout_$TAG.log
tail -n 20 gpurun_out/pytest_layout_$TAG.log
for c in c1 c4 c5; do for md in fp16 tf32; do
  timeout 600 python bench.py --config $c --mode $md --steps 50 --warmup 5 > gpurun_out/bench_${c}_${md}_$TAG.log 2>&1
  echo "== $c $md"; tail -c 400 gpurun_out/bench_${c}_${md}_$TAG.log; echo
done; done
