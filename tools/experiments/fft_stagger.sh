# A/B of the first-load stagger of the persistent FFT passes (FB_FFT_STAGGER ns per CTA slot)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/stagger.jsonl
for r in 1 2 3; do
for cfg in "" "FB_FFT_STAGGER=1" "FB_FFT_STAGGER=300" "FB_FFT_STAGGER=100"; do
env $cfg timeout 60 python tools/fft_pass_bench.py 2048 2048 100 | sed "s/}}/, \"cfg\": \"$cfg\"}}/" >> gpurun_out/stagger.jsonl 2>&1
done; done
for cfg in "" "FB_FFT_STAGGER=300"; do
env $cfg timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-extras | sed "s/^/$cfg /" >> gpurun_out/stagger.jsonl 2>&1
done
cat gpurun_out/stagger.jsonl
