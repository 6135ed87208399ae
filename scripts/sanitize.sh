#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the graph-replayed
# V-cycle and native GMRES (scripts/sanitize_run.py); logs into gpurun_out/.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for w in "C1 1 bench" "C5 10 bench" "C5 10 mcgs"; do
  set -- $w; tag=$1_$2_$3
  for tool in memcheck racecheck synccheck; do
    extra=""; [ $tool = memcheck ] && extra="--leak-check no"
    timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
        python scripts/sanitize_run.py $1 $2 $3 > gpurun_out/san_${tool}_${tag}.log 2>&1
    echo "$tool $tag rc=$?" | tee -a gpurun_out/san_summary.txt
    tail -3 gpurun_out/san_${tool}_${tag}.log >> gpurun_out/san_summary.txt
  done
done
