#!/bin/bash
# Interleaved bench comparison of prebuilt libraries abtmp/lib_<name>.so:
#   bash tools/ab_lib.sh TAG "old new [more ...]" [bench args]
# runs the names forward then backward, twice (ABBA for two names), one bench line each;
# the last name's library is left installed.
TAG=$1; NAMES=$2; shift 2
REV=$(echo $NAMES | tr ' ' '\n' | tac | tr '\n' ' ')
for rep in 1 2; do
  for v in $NAMES $REV; do
    cp abtmp/lib_$v.so paper_2308_15152_b200/libemusgemm.so
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-secondary "$@" 2>/dev/null | \
      python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', round(d['value'],2), round(d['ms_per_step']*1000,1), d['clocks']['sm_mhz'])"
  done
done > gpurun_out/ablib_$TAG.log
python - "$TAG" <<'EOF'
import sys, collections
d = collections.defaultdict(list)
for l in open(f"gpurun_out/ablib_{sys.argv[1]}.log"):
    p = l.split()
    if len(p) >= 2:
        d[p[0]].append(float(p[1]))
for k, v in d.items():
    print(f"{k:10s} mean {sum(v) / len(v):8.2f}  runs {v}")
EOF
