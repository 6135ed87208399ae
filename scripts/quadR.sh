run() { python bench.py --steps 10 --no-solve --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3))"; }
run quad-long-rows
CAMG_SELL_QUAD_BLOCKS=100000 run pair-only
run quad-long-rows
