#!/bin/bash
# launch list of one C3 V-cycle with the fused lambda side on every level, and
# one full ncu capture of the fused kernel
mkdir -p gpurun_out
export CAMG_LAM_FUSED=${CAMG_LAM_FUSED:-2}
cfg=${1:-C3}; sc=${2:-1}
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_lam_${cfg}.csv \
    python scripts/vc_launches.py $cfg $sc > gpurun_out/ncu_lam_${cfg}.log 2>&1
echo "list rc=$?"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_lam_ilu_cl -c 3 \
    -o gpurun_out/lam_full_${cfg} -f python scripts/vc_launches.py $cfg $sc > gpurun_out/ncu_lamfull_${cfg}.log 2>&1
echo "full rc=$?"
