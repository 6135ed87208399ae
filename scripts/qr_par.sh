run() { python scripts/setup_breakdown.py 1 > gpurun_out/qr_$1.log 2>&1; echo "$1 $(grep -o "'tentative_u': [0-9.]*" gpurun_out/qr_$1.log)"; }
run parallel
CAMG_QR_SERIAL=1 run serial
