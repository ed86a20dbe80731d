# A/B of the BF16 TMEM drain interval (FB_BF16_KP k-blocks of 64) + parity of each variant
cd $GRAFT_REPO_ROOT
P=paper_2004_09883_b200
rm -f gpurun_out/bf_kp.txt
for r in 1 2; do
for kp in 4 8 16; do
L=$P/libfb.so; [ $kp != 4 ] && L=$P/libfb_kp$kp.so
FB_LIB=$L timeout 300 python tools/bf16_bench.py | sed "s/}/, \"kp\": $kp}/" >> gpurun_out/bf_kp.txt 2>&1
done; done
for kp in 8 16; do FB_LIB=$P/libfb_kp$kp.so timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -k bf16 2>&1 | tail -1 | sed "s/^/kp=$kp /" >> gpurun_out/bf_kp.txt; done
cat gpurun_out/bf_kp.txt
