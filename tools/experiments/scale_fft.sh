cd $GRAFT_REPO_ROOT
for shp in "2048 2048" "4096 2048" "8192 2048" "2048 512" "8192 512"; do
  set -- $shp
  FLUSH=write+read timeout 60 python tools/fft_pass_bench.py $1 $2 5 > /dev/null 2>&1 && \
  FLUSH=write+read timeout 120 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/scale_$1_$2.csv python tools/fft_pass_bench.py $1 $2 5 > /dev/null 2>&1
done
