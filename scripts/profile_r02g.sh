#!/bin/bash
# Round-2 evidence after the uniform-slice loops and offset-aligned slots (run under gpurun from the repo root):
# (1) one-V-cycle ncu launch lists (gpu__time_duration + DRAM bytes, --clock-control none) for C5, C3, C2
# (2) one `ncu --set full` capture of the dominant kernel on C5: the fine-level Jacobi predictor sweep on
#     masked slots with shared value groups (k_sell_row<3,3,0,1,1,1,1>), the launch bench.py times for `roofline`
mkdir -p gpurun_out
for c in C5 C3 C2; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/r02g_vcycle_launches_${c}.csv \
      python scripts/vc_launches.py $c 1 > gpurun_out/r02g_ncu_vc_${c}.log 2>&1
  echo "$c list rc=$?"
done
CMD="python bench.py --steps 1 --warmup 3 --no-solve --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'k_sell_rowILi3ELi3ELb0ELb1ELi1ELb1ELb1E' -s 2 -c 1 \
    -o gpurun_out/r02g_dominant_kernel_c5 -f $CMD > gpurun_out/r02g_ncu_dom.log 2>&1
echo "dominant rc=$?"
