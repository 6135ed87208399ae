# C5 setup phases (setup_breakdown)
run() { python scripts/setup_breakdown.py 1 > gpurun_out/setup_$1.log 2>&1
  echo "$1 $(grep -o "'rap_K': [0-9.]*" gpurun_out/setup_$1.log)"; }
run lb64_16
