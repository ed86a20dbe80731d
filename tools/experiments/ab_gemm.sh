cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -m gpu -k "persistent or vs_oracle or variants" 2>&1 | tail -3
for r in 1 2; do
for sz in "4096 4096 4096 20" "8192 8192 8192 10" "16384 16384 16384 5" "32768 32768 32768 3"; do
for v in "FB_GEMM_PERSIST=0" "FB_GEMM_PERSIST=1"; do
  env $v timeout 300 python tools/gemm_bench.py $sz | VAR="$v" python -c "import json,os,sys; d=json.loads(sys.stdin.read()); print(d['m'], os.environ['VAR'], round(d['ms'],3), round(d['tflops'],1), d['rel_l2_vs_torch_f64'])"
done; done; done
