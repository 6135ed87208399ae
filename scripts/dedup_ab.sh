set -x
python -m pytest tests/test_gpu_parity.py -q -k "shared_value or masked_sell" 2>&1 | tail -5
python bench.py --no-cpu-baseline --rhs-seeds "" > gpurun_out/dd_on.log 2>gpurun_out/dd_on.err; tail -c 400 gpurun_out/dd_on.err
CAMG_SELL_DEDUP=0 python bench.py --no-cpu-baseline --rhs-seeds "" > gpurun_out/dd_off.log 2>gpurun_out/dd_off.err
python - <<'P'
import json
for f in ('dd_on','dd_off'):
    try:
        l=[x for x in open('gpurun_out/%s.log'%f) if x.startswith('{')][-1]; d=json.loads(l)
        print(f, d['ms_per_step'], d['roofline']['avg_launch_ms'], d['spmv']['ms'], d['solve']['time_to_solution_s'], d['solve']['gmres_iterations'], d['solve']['setup_s'], d['config']['device_memory_used_gb'])
    except Exception as e: print(f, 'ERR', e)
P
