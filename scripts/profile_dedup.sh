#!/bin/bash
# ncu --set full capture of the fine-level predictor pass with shared value groups (C5)
CMD="python bench.py --steps 1 --warmup 3 --no-solve --no-cpu-baseline"
$CMD > gpurun_out/plain_dd.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_sell_row -s 23 -c 1 \
    -o gpurun_out/prof_dd_c5 $CMD > gpurun_out/ncu_dd.log 2>&1
echo rc=$?
