# C5 time to solution for smoother variants (bench line fields), one GPU
for S in "$@"; do
  CAMG_BENCH_SMOOTHER=$S timeout 600 python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['solve']
print('$S', round(d['ms_per_step'],2), s['gmres_iterations'], s['converged'], round(s['time_to_solution_s'],3))" || echo "$S failed"
done
