#!/bin/bash
# grid cap of the one-lane-per-row SELL kernels (CAMG_SELL_CTAS x 148 x 4 CTAs of 64 threads): V-cycle / K pass / SpMV
run() { python bench.py --steps 10 --no-solve --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3), round(d['roofline']['avg_launch_ms'],4), round(d['spmv']['ms'],4))"; }
for c in "$@"; do CAMG_SELL_CTAS=$c run ctas=$c; done
