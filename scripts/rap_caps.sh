# C5 setup phases (setup_breakdown)
run() { CAMG_DEBUG=1 python scripts/setup_breakdown.py 1 > gpurun_out/setup_$1.log 2>&1
  echo "$1 $(grep -o "{'generate.*" gpurun_out/setup_$1.log)"; }
run default
