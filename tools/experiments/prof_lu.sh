cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras --only lu_f64_2048"
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --only lu_f64_2048 > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/lu_launches.csv -k regex:"lu_|gemm_f64" -c 3000 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --only lu_f64_2048 > /dev/null 2>&1
