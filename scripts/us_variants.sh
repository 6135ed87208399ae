#!/bin/bash
# V-cycle / K pass / SpMV of libcamg variants in paper_1912_09056_b200/ab (run under gpurun): us_variants.sh name[:USLICE] ...
run() { CAMG_SELL_USLICE=${2:-2} python bench.py --steps 10 --no-solve --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 uslice=${2:-2}', round(d['ms_per_step'],3), round(d['roofline']['avg_launch_ms'],4), round(d['spmv']['ms'],4))"; }
for a in "$@"; do
  v=${a%%:*}; m=2; [[ "$a" == *:* ]] && m=${a##*:}
  if [ "$v" == default ]; then run default $m; else CAMG_LIB=$PWD/paper_1912_09056_b200/ab/libcamg_$v.so run $v $m; fi
done
