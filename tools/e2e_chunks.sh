for rep in 1 2; do for c in 8 16 32 32 16 8; do
EMU_HOST_CHUNKS=$c timeout 300 python bench.py --no-cpu-baseline --no-secondary --steps 5 --warmup 3 --e2e-steps 10 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('chunks=$c', round(d['e2e']['value'],3))"
done; done
