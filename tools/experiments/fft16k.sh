cd $GRAFT_REPO_ROOT
timeout 120 python tools/fft_pass_bench.py 16384 16384 5 > gpurun_out/f16.json 2>&1 || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file gpurun_out/f16.csv python tools/fft_pass_bench.py 16384 16384 3 > /dev/null 2>&1
