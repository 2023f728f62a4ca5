#!/bin/bash
# Interleaved bench comparison of environment settings (tuning knobs) on one build:
#   bash tools/ab_env.sh TAG "A=1 B=2" "A=0" [...] -- [bench args]
# runs the settings forward then backward, twice; one bench line each.
TAG=$1; shift
VARS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do VARS+=("$1"); shift; done
[ "$1" = "--" ] && shift
ORDER=("${VARS[@]}")
for ((i=${#VARS[@]}-1; i>=0; i--)); do ORDER+=("${VARS[$i]}"); done
for rep in 1 2; do
  for v in "${ORDER[@]}"; do
    env $v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-secondary "$@" 2>/dev/null | \
      python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v'.replace(' ', ','), round(d['value'],2), round(d['ms_per_step']*1000,1), d['clocks']['sm_mhz'])"
  done
done > gpurun_out/abenv_$TAG.log
python - "$TAG" <<'PY'
import sys, collections
d = collections.defaultdict(list)
for l in open(f"gpurun_out/abenv_{sys.argv[1]}.log"):
    p = l.split()
    if len(p) >= 2:
        d[p[0]].append(float(p[1]))
for k, v in d.items():
    print(f"{k:40s} mean {sum(v) / len(v):8.2f}  runs {v}")
PY
