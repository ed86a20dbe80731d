# BF16 GEMM: persistent clusters (FB_BF16_PERSIST) and ring depth (libfb_s7.so: 7 stages), interleaved
cd $GRAFT_REPO_ROOT
P=paper_2004_09883_b200
for r in 1 2; do
  for v in "FB_BF16_PERSIST=0" "FB_BF16_PERSIST=1" "FB_BF16_PERSIST=0 FB_LIB=$P/libfb_s7.so" "FB_BF16_PERSIST=1 FB_LIB=$P/libfb_s7.so"; do
    env $v timeout 300 python tools/bf16_bench.py | VAR="$v" python -c "
import json, os, sys
for ln in sys.stdin:
    d = json.loads(ln); print(os.environ['VAR'].replace('$P/', ''), d['n'], round(d['ms'], 4), round(d['tflops']), 'cublas', round(d['cublas_ms'], 4))"
  done
done
