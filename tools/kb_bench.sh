run() { timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-secondary "$@" 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['value'],2), d['clocks']['sm_mhz'], '%.3g' % d['rel_frobenius_vs_fp64'], '%.3g' % d['max_rel_error_vs_fp64'])"; }
for rep in 1 2; do
echo "c2 fp16 kb64: $(run)"; echo "c2 fp16 kb128: $(run --kblock 128)"; echo "c2 fp16 kb256: $(run --kblock 256)"
echo "c2 tf32 kb64: $(run --mode tf32)"; echo "c2 tf32 kb128: $(run --mode tf32 --kblock 128)"
echo "c2 fp16 astat0: $(EMU_TS_ASTAT=0 run)"
done
