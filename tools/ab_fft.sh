cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab.jsonl
timeout 400 python -m pytest tests/test_fft_gpu.py tests/test_comm_gpu.py -m gpu -q -x 2>&1 | tail -1 > gpurun_out/ab_tests.log
for shp in "2048 2048" "256 256" "16384 16384"; do
  set -- $shp
  timeout 60 python tools/fft_pass_bench.py $1 $2 20 >> gpurun_out/ab.jsonl 2>&1
  FB_FFT_NO_PDL=1 timeout 60 python tools/fft_pass_bench.py $1 $2 20 >> gpurun_out/ab.jsonl 2>&1
done
timeout 200 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/b_pdl.json 2>&1
FB_FFT_NO_PDL=1 timeout 200 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/b_nopdl.json 2>&1
