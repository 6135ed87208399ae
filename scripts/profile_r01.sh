#!/bin/bash
# ncu evidence for round 1 (run under gpurun from the repo root)
set -x
CMD="python bench.py --scale 2 --steps 2 --warmup 3 --no-solve --no-cpu-baseline"
$CMD > gpurun_out/plain_s2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_s2.csv $CMD > gpurun_out/ncu_launches.log 2>&1
CMD5="python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline"
$CMD5 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_resid -s 40 -c 2 -o gpurun_out/prof_resid_c5 $CMD5 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
