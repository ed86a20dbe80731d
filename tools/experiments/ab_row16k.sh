# 16384-long row kernels: one CTA per line (FB_FFT_ROW16K=1) vs a CTA pair per line (=2, 2 or 3 CTAs/SM)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_fft_gpu.py tests/test_comm_gpu.py -x -q -m gpu -k "row16384 or 16384_rows or longrow" 2>&1 | tail -2
bash tools/ab_env.sh "FB_FFT_ROW16K=1|FB_FFT_ROW16K=2|FB_FFT_ROW16K=2 FB_FFT_ROW16K_CPS=3" "16384 16384;4096 16384" 3 2>&1 | tail -6
