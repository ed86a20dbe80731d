cd $GRAFT_REPO_ROOT
rm -f gpurun_out/sweep.jsonl
for cfg in "" "FB_FFT_COL_C=2" "FB_FFT_COL_C=8" "FB_FFT_COL_NB=2" "FB_FFT_ROW_NB=2" "FB_FFT_NO_PDL=1" "FB_FFT_PAIR=0" "FB_FFT_PAIR=0 FB_FFT_COL_C=4" "FB_FFT_PAIR_TMA=0"; do
env $cfg timeout 60 python tools/fft_pass_bench.py 2048 2048 40 | sed "s/}}/, \"cfg\": \"$cfg\"}}/" >> gpurun_out/sweep.jsonl 2>&1
done
