# A/B: column-pass outputs by direct stores (FB_FFT_COL_STG=1) vs X + TMA tensor store
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/colstg.jsonl
FB_FFT_COL_STG=1 timeout 900 python -m pytest tests/test_fft_gpu.py -m gpu -x -q > gpurun_out/colstg_tests.log 2>&1; tail -2 gpurun_out/colstg_tests.log
for r in 1 2 3; do
for cfg in "FB_FFT_COL_STG=0" "FB_FFT_COL_STG=1"; do
for n in "2048 2048" "1024 1024" "4096 4096" "512 512" "16384 16384"; do
env $cfg timeout 60 python tools/fft_pass_bench.py $n 100 | sed "s|}}|, \"cfg\": \"$cfg\"}}|" >> gpurun_out/colstg.jsonl 2>&1
done; done; done
