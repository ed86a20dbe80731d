# FFT 2048^2 probe: knob timings + one ncu --set full capture of the two passes (stall reasons)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/probe.jsonl
for cfg in "" "FB_FFT_ROW_NB=2" "FB_FFT_COL_NB=2" "FB_FFT_COL_C=8" "FB_FFT_COL_C=2" "FB_FFT_PAIR=0" "FLUSH=none"; do
env $cfg timeout 60 python tools/fft_pass_bench.py 2048 2048 60 | sed "s/}}/, \"cfg\": \"$cfg\"}}/" >> gpurun_out/probe.jsonl 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fft_pass" -s 20 -c 2 -o gpurun_out/probe_fft2048 python tools/fft_pass_bench.py 2048 2048 12 > gpurun_out/probe_ncu.log 2>&1
ncu -i gpurun_out/probe_fft2048.ncu-rep --page raw --csv > gpurun_out/probe_raw.csv 2>&1
ncu -i gpurun_out/probe_fft2048.ncu-rep --page source --csv --print-source sass > gpurun_out/probe_src.csv 2>&1
cat gpurun_out/probe.jsonl
