cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k bf16 2>&1 | tail -5 > gpurun_out/bf.log
FB_BF16_CLUSTER=2 timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k bf16 2>&1 | tail -2 >> gpurun_out/bf.log
timeout 300 python tools/bf16_bench.py > gpurun_out/bf_bench.txt 2>&1
FB_BF16_CLUSTER=2 timeout 300 python tools/bf16_bench.py >> gpurun_out/bf_bench.txt 2>&1
