#!/bin/bash
# bench lines of every config (C1-C4 with the reference-package CPU baseline alongside), then C5 and the reference arm
for c in C1 C2 C3 C4; do python bench.py --config $c > gpurun_out/r02g_bench_$c.log 2> gpurun_out/r02g_bench_$c.err; echo "$c rc=$?"; done
python bench.py > gpurun_out/r02g_bench_c5.log 2> gpurun_out/r02g_bench_c5.err; echo "C5 rc=$?"
python bench.py --impl reference > gpurun_out/r02g_reference_arm.log 2> gpurun_out/r02g_reference_arm.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?"
