python -m pytest tests/test_gpu_parity.py -q -k "shared_value or masked_sell or sell_block" 2>&1 | tail -2
run() { python bench.py --steps 10 --no-solve --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],3), round(d['roofline']['avg_launch_ms'],4), round(d['spmv']['ms'],4))"; }
run default
for v in ca; do CAMG_LIB=$PWD/paper_1912_09056_b200/ab/libcamg_$v.so run $v; done
