run() { python bench.py --steps 10 --no-solve --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3))"; }
CAMG_SELL_PAIR=5000 run pair5000
CAMG_SELL_PAIR=2000 run pair2000
CAMG_SELL_PAIR=8000 run pair8000
CAMG_SELL_PAIR=9000 run pair9000
CAMG_SELL_PAIR=5000 run pair5000
