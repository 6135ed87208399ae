#!/bin/bash
# launch lists (one V-cycle) of the smaller configs
mkdir -p gpurun_out
for c in "$@"; do
  cfg=${c%/*}; sc=${c#*/}; [ "$sc" = "$c" ] && sc=1
  timeout 600 python scripts/vc_launches.py $cfg $sc > gpurun_out/vc_${cfg}_${sc}.log 2>&1 || { echo "plain $c failed"; tail gpurun_out/vc_${cfg}_${sc}.log; continue; }
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/launches_${cfg}_${sc}.csv \
      python scripts/vc_launches.py $cfg $sc > gpurun_out/ncu_${cfg}_${sc}.log 2>&1
  echo "$c rc=$?"; cat gpurun_out/vc_${cfg}_${sc}.log | tail -1
done
