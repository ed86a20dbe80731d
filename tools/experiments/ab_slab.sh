cd $GRAFT_REPO_ROOT
rm -f gpurun_out/slab.jsonl
for n in "16384 16384" "2048 2048" "8192 8192"; do
timeout 120 python tools/slab_bench.py $n >> gpurun_out/slab.jsonl 2>&1
FB_SLAB_FUSED=0 timeout 120 python tools/slab_bench.py $n >> gpurun_out/slab.jsonl 2>&1
done
timeout 120 python tools/fft_pass_bench.py 16384 16384 10 >> gpurun_out/slab.jsonl 2>&1
