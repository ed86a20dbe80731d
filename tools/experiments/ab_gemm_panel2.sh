# FP32 GEMM N-panel width sweep (FB_GEMM_NPANEL), interleaved
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for sz in "8192 8192 8192 10" "16384 16384 16384 4" "32768 32768 32768 3" "32768 8192 32768 3"; do
for v in "FB_GEMM_NPANEL=0" "FB_GEMM_NPANEL=1024" "FB_GEMM_NPANEL=2048"; do
  env $v timeout 300 python tools/gemm_bench.py $sz | VAR="$v" python -c "import json,os,sys; d=json.loads(sys.stdin.read()); print(d['m'], d['n'], os.environ['VAR'], round(d['ms'],3), round(d['tflops'],1))"
done; done; done
