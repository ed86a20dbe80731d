# A/B: pair step with one lane exchange per element pair (FB_FFT_PAIR2=1) vs per element
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/pair2.jsonl
for r in 1 2 3 4 5 6; do
for cfg in "FB_FFT_PAIR2=0" "FB_FFT_PAIR2=1"; do
env $cfg timeout 60 python tools/fft_pass_bench.py 2048 2048 200 | sed "s|}}|, \"cfg\": \"$cfg\"}}|" >> gpurun_out/pair2.jsonl 2>&1
done; done
