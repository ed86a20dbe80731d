# BF16 GEMM (persistent): L2 rasterisation group size GROUP_M (libfb_gN.so builds), interleaved
cd $GRAFT_REPO_ROOT
P=paper_2004_09883_b200
for r in 1 2; do
  for L in libfb.so libfb_g2.so libfb_g4.so libfb_g16.so; do
    FB_LIB=$P/$L timeout 300 python tools/bf16_bench.py | L=$L python -c "
import json, os, sys
for ln in sys.stdin:
    d = json.loads(ln); print(os.environ['L'], d['n'], round(d['ms'], 4), round(d['tflops']))"
  done
done
