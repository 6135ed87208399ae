# V-cycle ms on C5 for the MC-SGS execution variants (no solve)
run() { python bench.py --steps 10 --no-solve --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3))"; }
run default
CAMG_PDL=0 run no-pdl
CAMG_MCGS_CTA=0 run no-cta
