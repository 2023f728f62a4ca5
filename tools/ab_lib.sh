#!/bin/bash
# ABBA bench comparison of two prebuilt libraries (abtmp/lib_old.so vs abtmp/lib_new.so):
#   bash tools/ab_lib.sh TAG [bench args]
TAG=$1; shift
for rep in 1 2; do
  for v in old new new old; do
    cp abtmp/lib_$v.so paper_2308_15152_b200/libemusgemm.so
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-secondary "$@" 2>/dev/null | \
      python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', round(d['value'],2), round(d['ms_per_step']*1000,1), d['clocks']['sm_mhz'])"
  done
done > gpurun_out/ablib_$TAG.log
cp abtmp/lib_new.so paper_2308_15152_b200/libemusgemm.so
