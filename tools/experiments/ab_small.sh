cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fft_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/small_tests.log
rm -f gpurun_out/small.txt
for cfg in "" "FB_FFT_SMALL=0"; do
env $cfg timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --only fft2d_256_fwd_inv > gpurun_out/s_x.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/s_x.json').read().strip().splitlines()[-1]); print('$cfg', d['blocks']['fft2d_256_fwd_inv']['ms_per_step'])" >> gpurun_out/small.txt
env $cfg timeout 60 python tools/fft_pass_bench.py 256 256 30 >> gpurun_out/small.txt 2>&1
env $cfg timeout 60 python tools/fft_pass_bench.py 64 128 30 >> gpurun_out/small.txt 2>&1
done
