for m in gpu host; do CAMG_TENTATIVE=$m python bench.py --no-cpu-baseline --no-solve --steps 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$m', d['ms_per_step'], [ (l['n_u'],l['nnz_K']) for l in d['config']['levels']])"; done
python scripts/setup_breakdown.py 2>&1 | tail -25
CAMG_TENTATIVE=gpu python scripts/setup_breakdown.py 2>&1 | tail -25
