#!/bin/bash
# full round check: tests, smoke, bench (ours + reference), ncu launch list + captures.  bash tools/gpu_round.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
python paper_2308_15152_b200/build.py > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1
timeout 600 python bench.py --mode tf32 > gpurun_out/bench_default_tf32_$TAG.log 2>&1
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/bench_c3_fp16_$TAG.log 2>&1
timeout 600 python bench.py --config c3 --mode tf32 --steps 20 --warmup 3 > gpurun_out/bench_c3_tf32_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 10 --csv --log-file gpurun_out/launches_c2_fp16_$TAG.csv python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c2_fp16_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c2_tf32_$TAG python bench.py --mode tf32 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c3_fp16_$TAG python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# raw-page exports travel back; the full reports only while gpurun_out stays under its 64 MiB cap
for r in gpurun_out/prof_*_$TAG.ncu-rep; do ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null; done
for r in gpurun_out/prof_c2_tf32_$TAG.ncu-rep gpurun_out/prof_c3_fp16_$TAG.ncu-rep; do
  [ $(du -sm gpurun_out | cut -f1) -gt 48 ] && rm -f $r
done
rm -f gpurun_out/tc_samples.npz
du -sh gpurun_out
echo done
