# A/B: column-pass last stage on column pairs with 16-byte shared accesses (FB_FFT_COLPAIR=1)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/colpair.jsonl
timeout 900 python -m pytest tests/test_fft_gpu.py -m gpu -x -q -k "bitwise or variants" > gpurun_out/colpair_tests.log 2>&1; tail -2 gpurun_out/colpair_tests.log
FB_FFT_COLPAIR=1 timeout 900 python -m pytest tests/test_fft_gpu.py tests/test_comm_gpu.py -m gpu -x -q > gpurun_out/colpair_tests2.log 2>&1; tail -2 gpurun_out/colpair_tests2.log
for r in 1 2 3 4; do
for cfg in "FB_FFT_COLPAIR=0" "FB_FFT_COLPAIR=1"; do
for n in "2048 2048" "1024 1024" "512 512" "4096 4096"; do
env $cfg timeout 60 python tools/fft_pass_bench.py $n 200 | sed "s|}}|, \"cfg\": \"$cfg\"}}|" >> gpurun_out/colpair.jsonl 2>&1
done; done; done
