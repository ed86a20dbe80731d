cd $GRAFT_REPO_ROOT
for v in "X=0" "FB_FFT_NO_TMA_COL=1" "FB_FFT_NO_TMA_ROW=1" "FB_FFT_NO_TMA=1"; do
  echo "== $v" >> gpurun_out/race.log
  for i in 1 2; do env $v timeout 300 python -m pytest tests/test_fft_gpu.py -m gpu -q -k "deterministic or 16384 or four_step" 2>&1 | tail -1 >> gpurun_out/race.log; done
done
