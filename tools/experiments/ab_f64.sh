cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k f64 2>&1 | tail -1 > gpurun_out/ab_f64.log
for c in 0 3 4 5 6; do FB_F64_CFG=$c timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --only gemm_f64_2048 > gpurun_out/bf64_$c.json 2>&1; done
