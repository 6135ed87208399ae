run() { python bench.py --steps 10 --no-solve --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3))"; }
run default
CAMG_MCGS_CTA_G=8 run g8
CAMG_MCGS_CTA_G=4 run g4
CAMG_MCGS_CTA_G=16 run g16
CAMG_MCGS_CTA=0 run no-cta
