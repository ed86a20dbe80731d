# ncu --set full of the 2048^2 FFT passes (pair plan) for the row-pass investigation
cd $GRAFT_REPO_ROOT
timeout 60 python tools/fft_pass_bench.py 2048 2048 3 > gpurun_out/pr.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fft_pass" -s 4 -c 2 -o gpurun_out/fftrow python tools/fft_pass_bench.py 2048 2048 3 > gpurun_out/fftrow.log 2>&1
FB_FFT_PAIR=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fft_pass" -s 4 -c 2 -o gpurun_out/fftrow0 python tools/fft_pass_bench.py 2048 2048 3 > gpurun_out/fftrow0.log 2>&1
