cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab.jsonl
FB_FFT_COL_MAX_LOG2=10 timeout 400 python -m pytest tests/test_fft_gpu.py -m gpu -q -x 2>&1 | tail -1 > gpurun_out/ab_tests.log
timeout 60 python tools/fft_pass_bench.py 2048 2048 30 >> gpurun_out/ab.jsonl 2>&1
for lb in 4 5 6 7; do FB_FFT_COL_MAX_LOG2=10 FB_FFT_4STEP_LB=$lb timeout 60 python tools/fft_pass_bench.py 2048 2048 30 >> gpurun_out/ab.jsonl 2>&1; done
for lb in 6 7 8; do FB_FFT_4STEP_LB=$lb timeout 60 python tools/fft_pass_bench.py 16384 16384 10 >> gpurun_out/ab.jsonl 2>&1; done
FB_FFT_COL_MAX_LOG2=10 timeout 60 python tools/fft_pass_bench.py 2048 2048 5 > /dev/null 2>&1 && FB_FFT_COL_MAX_LOG2=10 timeout 120 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/nc_4s.csv python tools/fft_pass_bench.py 2048 2048 5 > /dev/null 2>&1
