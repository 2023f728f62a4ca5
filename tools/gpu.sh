#!/bin/bash
# One entry point for the GPU-box jobs of this repo (run through gpurun, from the
# repo root; everything lands in gpurun_out/):
#
#   bash tools/gpu.sh round TAG    build, GPU tests, smoke, bench (ours + reference),
#                                  ncu launch list of the bench command, ncu --set full
#                                  captures of the c2 fp16 / c2 tf32 / c3 fp16 kernels
#   bash tools/gpu.sh tests TAG    build, GPU tests, smoke
#   bash tools/gpu.sh ncu TAG      only the ncu launch list + captures
#   bash tools/gpu.sh ab TAG "ENV=a" "ENV=b" [bench args]
#                                  ABBA bench comparison of two environment settings
#                                  (tuning knobs such as EMU_PDL, EMU_GROUP_M, EMU_TS_N)
#   bash tools/gpu.sh probe TAG    the standalone tcgen05 probe tests (samples for tools/tc_fit.py)
set -u
CMD=${1:-round}
TAG=${2:-r}
mkdir -p gpurun_out
build() {
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
}
tests() {
  timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
}
ncu_all() {
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 20 --csv \
    --log-file gpurun_out/launches_c2_fp16_$TAG.csv python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-e2e --no-secondary > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c2_fp16_$TAG \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c2_tf32_$TAG \
    python bench.py --mode tf32 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:emu_sgemm -s 3 -c 1 -o gpurun_out/prof_c3_fp16_$TAG \
    python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  for r in gpurun_out/prof_*_$TAG.ncu-rep; do ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null; done
  for r in gpurun_out/prof_c2_tf32_$TAG.ncu-rep gpurun_out/prof_c3_fp16_$TAG.ncu-rep; do
    [ $(du -sm gpurun_out | cut -f1) -gt 48 ] && rm -f $r
  done
}
case $CMD in
  round)
    build; tests
    timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1
    timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1
    ncu_all ;;
  tests) build; tests ;;
  ncu) build; ncu_all ;;
  probe) build; timeout 600 python -m pytest tests/test_gpu_tcprobe.py -q > gpurun_out/probe_$TAG.log 2>&1 ;;
  ab)
    A=$3; B=$4; shift 4
    build
    for rep in 1 2; do
      for e in "$A" "$B" "$B" "$A"; do
        env $e timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-secondary "$@" 2>/dev/null | \
          python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$e', round(d['value'],2), d['clocks']['sm_mhz'])"
      done
    done > gpurun_out/ab_$TAG.log ;;
  *) echo "unknown command $CMD"; exit 2 ;;
esac
du -sh gpurun_out
echo done
