cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab.jsonl
timeout 900 python -m pytest tests/test_fft_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ab_tests.log
for n in "2048 2048" "1024 1024" "256 256" "4096 4096" "16384 16384"; do
timeout 60 python tools/fft_pass_bench.py $n 40 >> gpurun_out/ab.jsonl 2>&1
FB_LIB=paper_2004_09883_b200/libfb_old.so timeout 60 python tools/fft_pass_bench.py $n 40 | sed 's/}}/, "lib": "old"}}/' >> gpurun_out/ab.jsonl 2>&1
timeout 60 python tools/fft_pass_bench.py $n 40 >> gpurun_out/ab.jsonl 2>&1
done
