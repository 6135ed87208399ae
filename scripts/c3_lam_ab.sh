#!/bin/bash
# C3 (latency-bound) V-cycle with the lambda-side modes: CAMG_LAM_FUSED 1 (default) / 2 / 3, dense-inverse limit
run() { python bench.py --config ${CFG:-C3} --steps 50 --no-solve --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), d['vcycle_roofline']['kernels_per_cycle'])"; }
run default
CAMG_LAM_FUSED=2 run fused2
CAMG_LAM_FUSED=3 run fused3
CAMG_OVERLAP=0 run no-overlap
CAMG_OVERLAP=0 CAMG_LAM_FUSED=2 run no-overlap-fused2
CAMG_OVERLAP=0 CAMG_ILU_DENSE_MAX=16384 run no-overlap-dense16k
CAMG_ILU_DENSE_MAX=16384 run dense16k
