#!/bin/bash
# c3 (16384^3) tile-order / L2-policy sweep: DRAM bytes and duration of one launch (ncu,
# clocks not locked), optionally a bench value.  Entries: "EMU_TS_CLC EMU_GROUP_M EMU_L2_POLICY"
# (policy bits: 1 B evict_first, 2 A evict_last, 16 B evict_last).
#   bash tools/c3_raster.sh MODE BENCH "cfg1" "cfg2" ... > gpurun_out/c3_raster.log
MODE=$1; BENCH=$2; shift 2
for cfg in "$@"; do
  set -- $cfg
  export EMU_TS_CLC=$1 EMU_GROUP_M=$2 EMU_L2_POLICY=$3
  v=""
  if [ "$BENCH" = 1 ]; then
    v=$(timeout 300 python bench.py --config c3 --mode $MODE --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['value'],1), d['clocks']['sm_mhz'])")
  fi
  timeout 300 ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:emu_sgemm -s 2 -c 1 --csv python bench.py --config c3 --mode $MODE --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/n.csv 2>/dev/null
  d=$(grep -E "dram__bytes_read.sum|gpu__time" /tmp/n.csv | awk -F'","' '{print $(NF-2), $(NF)}' | tr -d '"' | tr '\n' ' ')
  echo "clc=$1 group=$2 pol=$3 bench(TF MHz): $v ncu: $d"
done
