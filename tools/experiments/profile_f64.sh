cd $GRAFT_REPO_ROOT
CMD2="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --only gemm_f64_2048"
timeout 300 $CMD2 > gpurun_out/b_g.json 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64" -s 1 -c 1 -o gpurun_out/r1_f64 $CMD2 > gpurun_out/r1_f64.log 2>&1
