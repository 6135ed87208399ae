# time to solution for smoother variants on one BASELINE config: config_sweep.sh C2 "kind,alpha,outer,pk,ps,pd,ck,cs,cd" ...
C=$1; shift
for S in "$@"; do
  CAMG_BENCH_SMOOTHER=$S timeout 900 python bench.py --config $C --steps 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['solve']
print('$C', '$S', round(d['ms_per_step'],3), s['gmres_iterations'], s['converged'], round(s['time_to_solution_s'],3))" || echo "$C $S failed"
done
