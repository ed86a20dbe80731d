# non-power-of-two 2D FFT: mixed-radix Stockham (FB_FFT_MIXED=1) vs Bluestein (=0)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fft_gpu.py -x -q -m gpu -k "non_power" 2>&1 | tail -2
bash tools/ab_env.sh "FB_FFT_MIXED=1|FB_FFT_MIXED=0" "1000 1000;2000 3000;360 480;2187 2187;1000 8000" 2 2>&1 | tail -10
