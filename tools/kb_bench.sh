#!/bin/bash
# Throughput and accuracy vs the combine interval KB (bench --kblock), interleaved, on the GPU box:
#   bash tools/kb_bench.sh [bench args]      e.g.  --config c3   or   --mode tf32
# prints one line per run: KB (0 = the default rule, R#7), TFlop/s, SM MHz, rel-Frobenius vs FP64
run() { timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-secondary "$@" 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['value'],2), d['clocks']['sm_mhz'], '%.3g' % d['rel_frobenius_vs_fp64'])"; }
for rep in 1 2; do
  for kb in 0 128 256 256 128 0; do
    a=""; [ $kb != 0 ] && a="--kblock $kb"
    echo "kb=$kb $(run "$@" $a)"
  done
done
