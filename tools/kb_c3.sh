for rep in 1 2; do for kb in 0 256 512 256 0; do
  a=""; [ $kb != 0 ] && a="--kblock $kb"
  timeout 300 python bench.py --config c3 --steps 10 --warmup 2 --no-cpu-baseline --no-e2e $a 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('kb=$kb', round(d['value'],1), d['clocks']['sm_mhz'], '%.3g' % d['rel_frobenius_vs_fp64'])"
done; done
