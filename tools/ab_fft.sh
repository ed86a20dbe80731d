cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab.jsonl
FB_FFT_ROW_NB=0 timeout 900 python -m pytest tests/test_fft_gpu.py -m gpu -q -x -k "pair or full_oracle or determin" 2>&1 | tail -3 > gpurun_out/ab_tests.log
for n in "2048 2048" "1024 1024" "2048 1024" "512 512"; do
timeout 60 python tools/fft_pass_bench.py $n 40 >> gpurun_out/ab.jsonl 2>&1
FB_FFT_ROW_NB=0 timeout 60 python tools/fft_pass_bench.py $n 40 >> gpurun_out/ab.jsonl 2>&1
done
FB_FFT_ROW_NB=0 timeout 120 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/pair.csv python tools/fft_pass_bench.py 2048 2048 3 > /dev/null 2>&1
