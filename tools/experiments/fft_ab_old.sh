# interleaved A/B of libfb_old.so (previous commit) vs the current build with knob settings
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/abold.jsonl
for r in 1 2 3 4; do
for cfg in "FB_LIB=paper_2004_09883_b200/libfb_old.so" "FB_FFT_STAGGER=0" "FB_FFT_STAGGER=300" "FB_FFT_L2PF=1" "FB_FFT_L2PF=1 FB_FFT_STAGGER=0"; do
env $cfg timeout 60 python tools/fft_pass_bench.py 2048 2048 150 | sed "s|}}|, \"cfg\": \"$cfg\"}}|" >> gpurun_out/abold.jsonl 2>&1
done; done
