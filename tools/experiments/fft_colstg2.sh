# verify the auto column-output rule (direct stores for C = 16 column passes)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/colstg2.jsonl
timeout 900 python -m pytest tests/test_fft_gpu.py tests/test_comm_gpu.py -m gpu -x -q > gpurun_out/colstg2_tests.log 2>&1; tail -2 gpurun_out/colstg2_tests.log
for r in 1 2; do
for cfg in "FB_FFT_COL_STG=0" "FB_FFT_COL_STG=-1"; do
for n in "2048 2048" "512 512" "256 256" "16384 16384" "8192 8192"; do
env $cfg timeout 60 python tools/fft_pass_bench.py $n 100 | sed "s|}}|, \"cfg\": \"$cfg\"}}|" >> gpurun_out/colstg2.jsonl 2>&1
done; done; done
