#!/bin/bash
# A/B of the uniform-slice loop on C5 (run under gpurun from the repo root): the new parity test, then the bench
# line (K pass, SpMV, V-cycle, GMRES) with the loop off and on
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "uniform_slice or shared_value or masked_sell" > gpurun_out/uslice_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/uslice_tests.log
for m in 1 2; do
  CAMG_SELL_USLICE=$m python bench.py --no-cpu-baseline --rhs-seeds "" > gpurun_out/uslice_bench_$m.log 2>&1
  echo "bench $m rc=$?"
  tail -1 gpurun_out/uslice_bench_$m.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms_per_step',d['ms_per_step'],'K pass ms',d['roofline']['avg_launch_ms'],'spmv ms',d['spmv']['ms'],'gmres',d['solve']['gmres_iterations'],d['solve']['time_to_solution_s'],'setup',d['solve']['setup_s'])"
done
