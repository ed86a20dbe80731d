# Profiles committed under profiles/ (run under gpurun; one GPU).
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --only gemm_f32_2048,gemm_f64_2048"
timeout 300 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv $CMD > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_pass|gemm_3xtf32|gemm_f64|split_" -s 0 -c 8 -o gpurun_out/r1_full $CMD > gpurun_out/r1_full.log 2>&1
