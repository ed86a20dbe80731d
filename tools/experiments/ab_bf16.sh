cd $GRAFT_REPO_ROOT
P=paper_2004_09883_b200
timeout 300 python tools/bf16_bench.py > gpurun_out/bf_bench.txt 2>&1
for g in 16 32; do FB_LIB=$P/libfb_g$g.so timeout 300 python tools/bf16_bench.py | sed "s/}/, \"group\": $g}/" >> gpurun_out/bf_bench.txt 2>&1; done
