#!/bin/bash
# ncu --set full of the fine-level predictor pass with the uniform-slice loop in mode $1 (run under gpurun)
mkdir -p gpurun_out
for m in "$@"; do
CMD="python bench.py --steps 1 --warmup 3 --no-solve --no-cpu-baseline"
CAMG_SELL_USLICE=$m timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'k_sell_rowILi3ELi3ELb0ELb1ELi1ELb1ELb1E' -s 2 -c 1 \
    -o gpurun_out/r02d_dominant_uslice$m -f $CMD > gpurun_out/r02d_ncu_dom_$m.log 2>&1
echo "mode $m rc=$?"
done
