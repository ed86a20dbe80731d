# Profiles committed under profiles/ (run under gpurun; one GPU).  Every ncu command below is
# preceded by the same command run without ncu (exit 0).
cd $GRAFT_REPO_ROOT
R=${R:-r2}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv $CMD > /dev/null 2>&1
HCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras"
timeout 600 $HCMD > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_pass|fft_col1024" -s 10 -c 2 -o gpurun_out/${R}_fft2048 $HCMD > gpurun_out/${R}_fft2048.log 2>&1
GCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --only gemm_f32_2048,gemm_f64_2048,lu_f64_2048"
timeout 600 $GCMD > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_3xtf32|split_both" -s 2 -c 2 -o gpurun_out/${R}_gemm $GCMD > gpurun_out/${R}_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64_dmma" -s 1 -c 1 -o gpurun_out/${R}_f64 $GCMD > gpurun_out/${R}_f64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lu_panel_tma|lu_rank|lu_swap" -s 60 -c 3 -o gpurun_out/${R}_lu $GCMD > gpurun_out/${R}_lu.log 2>&1
BCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --only gemm_bf16_8192,fft2d_16384"
timeout 600 $BCMD > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_pair" -s 2 -c 1 -o gpurun_out/${R}_bf16 $BCMD > gpurun_out/${R}_bf16.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_row16384|fft_pass_tma_kernel<7" -s 3 -c 3 -o gpurun_out/${R}_fft16k $BCMD > gpurun_out/${R}_fft16k.log 2>&1
