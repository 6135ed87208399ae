#!/bin/bash
# per-kernel launch list of the C5 V-cycle (kernels that only run in the solve phase)
CMD="python bench.py --steps 1 --warmup 3 --no-solve --no-cpu-baseline"
$CMD > gpurun_out/plain_vc.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_sell_row|k_resid|k_jacobi|k_spmv|k_lam|k_corr|k_lu_solve|k_b1_correct' -c 3000 --csv \
    --log-file gpurun_out/launches_vc_c5.csv $CMD > gpurun_out/ncu_vc.log 2>&1
echo rc=$?
