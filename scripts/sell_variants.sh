run() { python bench.py --steps 10 --no-solve --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3))"; }
run quad-default
CAMG_SELL_QUAD=0 run pair
