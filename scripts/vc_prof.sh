# V-cycle timing + GMRES + one-cycle kernel breakdown (ncu launch list) on C5
CMD="python bench.py --steps 1 --warmup 3 --no-solve --no-cpu-baseline"
python bench.py --steps 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['ms_per_step'], d['solve']['gmres_iterations'], d['solve']['time_to_solution_s'], d['solve']['setup_s'])
"
[ "$1" = "noprof" ] && exit 0
$CMD > gpurun_out/plain_vc.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_sell|k_resid|k_jacobi|k_spmv|k_lam|k_corr|k_lu_solve|k_b1|k_mcgs|k_ilu|k_copy|k_gs|k_pred' -c 3000 --csv \
    --log-file gpurun_out/vc_launches.csv $CMD > gpurun_out/ncu_vc.log 2>&1
python scripts/launch_breakdown.py gpurun_out/vc_launches.csv > gpurun_out/vc_breakdown.txt
head -22 gpurun_out/vc_breakdown.txt
