cd $GRAFT_REPO_ROOT
rm -f gpurun_out/sweep.jsonl
for cfg in "" "FB_FFT_GRID_WAVES=3" "FB_FFT_GRID_WAVES=4" "FB_FFT_GRID_WAVES=3 FB_FFT_COL_NB=2 FB_FFT_ROW_NB=2"; do
env $cfg timeout 60 python tools/fft_pass_bench.py 2048 2048 40 | sed "s/}}/, \"cfg\": \"$cfg\"}}/" >> gpurun_out/sweep.jsonl 2>&1
env $cfg timeout 60 python tools/fft_pass_bench.py 16384 16384 10 | sed "s/}}/, \"cfg\": \"$cfg\"}}/" >> gpurun_out/sweep.jsonl 2>&1
done
