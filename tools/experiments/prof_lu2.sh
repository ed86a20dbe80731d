cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --only lu_f64_2048"
timeout 300 $CMD > /dev/null 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"lu_panel" -s 30 -c 2 -o gpurun_out/lu_panel $CMD > gpurun_out/r1_lu.log 2>&1
