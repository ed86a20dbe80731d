cd $GRAFT_REPO_ROOT
rm -f gpurun_out/ab.jsonl
for shp in "2048 2048" "16384 16384" "256 256" "8192 2048"; do
  set -- $shp
  FLUSH=write+read timeout 60 python tools/fft_pass_bench.py $1 $2 20 >> gpurun_out/ab.jsonl 2>&1
  FLUSH=write+read FB_FFT_NO_TMA_COL=1 timeout 60 python tools/fft_pass_bench.py $1 $2 20 >> gpurun_out/ab.jsonl 2>&1
done
FLUSH=write+read FB_FFT_COL_C=4 timeout 60 python tools/fft_pass_bench.py 2048 2048 20 >> gpurun_out/ab.jsonl 2>&1
FLUSH=write+read FB_FFT_COL_C=8 timeout 60 python tools/fft_pass_bench.py 16384 16384 10 >> gpurun_out/ab.jsonl 2>&1
