# A/B: split staging (FB_FFT_ROW_NB=0, 4 CTAs/SM) for the pair row pass, x first-load stagger
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/split.jsonl
FB_FFT_ROW_NB=0 timeout 600 python -m pytest tests/test_fft_gpu.py -m gpu -x -q -k "2048 or 1024 or 512 or pair or determin" > gpurun_out/split_tests.log 2>&1; tail -2 gpurun_out/split_tests.log
for r in 1 2 3; do
for cfg in "FB_FFT_STAGGER=0" "FB_FFT_STAGGER=300" "FB_FFT_ROW_NB=0 FB_FFT_STAGGER=0" "FB_FFT_ROW_NB=0 FB_FFT_STAGGER=300" "FB_FFT_ROW_NB=0 FB_FFT_STAGGER=150"; do
for n in "2048 2048" "1024 1024"; do
env $cfg timeout 60 python tools/fft_pass_bench.py $n 100 | sed "s/}}/, \"cfg\": \"$cfg\"}}/" >> gpurun_out/split.jsonl 2>&1
done; done; done
