# time decomposition of the 2048^2 passes (FB_FFT_DEBUG: 1 skip stages, 2 skip loads, 4 skip stores)
cd $GRAFT_REPO_ROOT
N=${N:-2048 2048}
for d in 0 1 2 4 6 5 3; do
FB_FFT_DEBUG=$d timeout 120 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/decomp_$d.csv python tools/fft_pass_bench.py $N 5 > /dev/null 2>&1
done
