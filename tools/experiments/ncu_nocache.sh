cd $GRAFT_REPO_ROOT
FLUSH=write+read timeout 60 python tools/fft_pass_bench.py 2048 2048 5 > /dev/null 2>&1 && \
FLUSH=write+read timeout 120 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/nc_2048.csv python tools/fft_pass_bench.py 2048 2048 5 > /dev/null 2>&1
FLUSH=write+read FB_FFT_NO_TMA=1 timeout 120 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/nc_2048_notma.csv python tools/fft_pass_bench.py 2048 2048 5 > /dev/null 2>&1
