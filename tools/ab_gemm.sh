cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_comm_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gemm_tests.log
rm -f gpurun_out/gemm_ab.txt
for cfg in "" "FB_GEMM_SPLIT2=1"; do
env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --only gemm_f32_2048 > gpurun_out/g_x.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g_x.json').read().strip().splitlines()[-1]); b=d['blocks']['gemm_f32_2048']; print('$cfg', b['ms_per_step'], b['value'], b['roofline']['kernel_ms'])" >> gpurun_out/gemm_ab.txt
done
