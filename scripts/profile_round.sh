#!/bin/bash
# ncu evidence on C5 for the current build (run under gpurun from the repo root):
# (0) the default bench line (no profiler)
# (1) per-kernel launch list of the V-cycle kernels (gpu__time_duration + DRAM bytes)
# (2) one `ncu --set full` capture of the dominant kernel: the fine-level
#     Jacobi predictor sweep on masked slots, k_sell_row<3, 3, 0, 1, 1, 1>
#     (selected by its mangled name)
TAG=${1:-r01}
python bench.py > gpurun_out/${TAG}_bench_c5.log 2>&1 || { echo bench failed; exit 1; }
CMD="python bench.py --steps 1 --warmup 3 --no-solve --no-cpu-baseline"
$CMD > gpurun_out/plain_dom.log 2>&1 || { echo plain failed; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_sell|k_resid|k_jacobi|k_spmv|k_lam|k_corr|k_lu_solve|k_b1_correct|k_mcgs|k_ilu|k_copy|k_add' -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches_vc_c5.csv $CMD > gpurun_out/ncu_vc.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'k_sell_rowILi3ELi3ELb0ELb1ELi1ELb1E' -s 2 -c 1 \
    -o gpurun_out/${TAG}_dominant_kernel_c5 $CMD > gpurun_out/ncu_dom.log 2>&1
echo rc=$?
