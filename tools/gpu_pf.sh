#!/bin/bash
python paper_2308_15152_b200/build.py > /dev/null 2>&1
for pf in 0 4 8 16 32; do
  EMU_PREFETCH=$pf timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_pf$pf.log 2>&1
  EMU_PREFETCH=$pf timeout 300 python bench.py --steps 300 --warmup 10 --mode tf32 --no-cpu-baseline --no-e2e > gpurun_out/bench_pf${pf}_tf32.log 2>&1
done
EMU_KERNEL=single timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_single.log 2>&1
