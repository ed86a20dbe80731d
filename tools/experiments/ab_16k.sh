cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fft_gpu.py tests/test_comm_gpu.py -m gpu -q -x -k "16384 or sampled or slab or fused" 2>&1 | tail -3 > gpurun_out/16k_tests.log
rm -f gpurun_out/16k.txt
for cfg in "" "FB_FFT_LONGROW=0"; do
env $cfg timeout 120 python tools/fft_pass_bench.py 16384 16384 10 >> gpurun_out/16k.txt 2>&1
env $cfg timeout 120 python tools/fft_pass_bench.py 1024 16384 20 >> gpurun_out/16k.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/f16.csv python tools/fft_pass_bench.py 16384 16384 3 > /dev/null 2>&1
