cd $GRAFT_REPO_ROOT
rm -f gpurun_out/sweep.jsonl
for cfg in "" "FB_FFT_COL_MAX_LOG2=10" "FB_FFT_COL_MAX_LOG2=10 FB_FFT_4STEP_LB=4" "FB_FFT_COL_MAX_LOG2=10 FB_FFT_4STEP_LB=5" "FB_FFT_COL_MAX_LOG2=10 FB_FFT_4STEP_LB=7" "FB_FFT_COL_MAX_LOG2=10 FB_FFT_4STEP_LB=3"; do
env $cfg timeout 60 python tools/fft_pass_bench.py 2048 2048 40 | sed "s/}}/, \"cfg\": \"$cfg\"}}/" >> gpurun_out/sweep.jsonl 2>&1
done
FB_FFT_COL_MAX_LOG2=10 FB_FFT_4STEP_LB=5 timeout 120 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/fs.csv python tools/fft_pass_bench.py 2048 2048 3 > /dev/null 2>&1
