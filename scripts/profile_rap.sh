#!/bin/bash
# ncu full capture of the Galerkin triple-product kernel (count pass) at C5/2
CMD="python scripts/setup_breakdown.py 2"
$CMD > gpurun_out/plain_rap.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_triple -c 1 \
    -o gpurun_out/prof_rap $CMD > gpurun_out/ncu_rap.log 2>&1
echo rc=$?
