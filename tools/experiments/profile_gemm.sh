cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --only gemm_f32_2048,gemm_f64_2048"
timeout 300 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_3xtf32|gemm_f64|split_" -s 4 -c 4 -o gpurun_out/r1_gemm $CMD > gpurun_out/r1_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --replay-mode application --import-source on -k regex:"fft_pass" -s 4 -c 2 -o gpurun_out/r1_fft_app $CMD > gpurun_out/r1_fft_app.log 2>&1
