#!/bin/bash
# offset-aligned slots A/B on C5 (run under gpurun): parity tests, then bench lines with CAMG_SELL_ALIGN=0 / 1
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "uniform_slice or shared_value or masked_sell or sell_block" > gpurun_out/align_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/align_tests.log
for m in 0 1; do
  CAMG_SELL_ALIGN=$m python bench.py --no-cpu-baseline --rhs-seeds "" > gpurun_out/align_bench_$m.log 2>&1
  echo "bench align=$m rc=$?"
  tail -1 gpurun_out/align_bench_$m.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms_per_step',d['ms_per_step'],'K pass ms',d['roofline']['avg_launch_ms'],'spmv ms',d['spmv']['ms'],'gmres',d['solve']['gmres_iterations'],d['solve']['time_to_solution_s'],'setup',d['solve']['setup_s'],d['solve']['setup_breakdown_s'], 'mem', d['config']['device_memory_used_gb'])"
done
