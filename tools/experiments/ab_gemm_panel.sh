# FP32 GEMM: one launch vs N-column panel launches (FB_GEMM_NPANEL) vs an in-kernel panel raster
# (FB_GEMM_RASTER_PANEL, tile columns per panel), interleaved
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for sz in "16384 16384 16384 4" "32768 32768 32768 3"; do
for v in "FB_GEMM_NPANEL=0" "FB_GEMM_NPANEL=4096" "FB_GEMM_NPANEL=2048" "FB_GEMM_RASTER_PANEL=16" "FB_GEMM_RASTER_PANEL=8" "FB_GEMM_RASTER_PANEL=32"; do
  env $v timeout 300 python tools/gemm_bench.py $sz | VAR="$v" python -c "import json,os,sys; d=json.loads(sys.stdin.read()); print(d['m'], os.environ['VAR'], round(d['ms'],3), round(d['tflops'],1), d['rel_l2_vs_torch_f64'])"
done; done; done
