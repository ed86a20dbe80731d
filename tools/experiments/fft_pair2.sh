# A/B: pair step variants (FB_FFT_PAIR2: 0 lane exchange per element, 1 per element pair,
# 2 last row stage fused with the pair step, no lane exchange)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/pair2.jsonl
timeout 900 python -m pytest tests/test_fft_gpu.py -m gpu -x -q -k "bitwise or variants or pair" > gpurun_out/pair2_tests.log 2>&1; tail -2 gpurun_out/pair2_tests.log
for r in 1 2 3 4; do
for cfg in "FB_FFT_PAIR2=1" "FB_FFT_PAIR2=2"; do
for n in "2048 2048" "1024 1024" "512 512"; do
env $cfg timeout 60 python tools/fft_pass_bench.py $n 200 | sed "s|}}|, \"cfg\": \"$cfg\"}}|" >> gpurun_out/pair2.jsonl 2>&1
done; done; done
