# configs[0]: 256x256 as one cluster kernel (FB_FFT_SMALL=8/16) vs the two-pass path (=0)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_fft_gpu.py -x -q -m gpu -k "256 or fourn or host" 2>&1 | tail -2
bash tools/ab_env.sh "FB_FFT_SMALL=0|FB_FFT_SMALL=8|FB_FFT_SMALL=16" "256 256" 3 2>&1 | tail -4
for v in 0 8 16; do FB_FFT_SMALL=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --only fft2d_256_fwd_inv 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('SMALL=$v', d['blocks']['fft2d_256_fwd_inv']['ms_per_step'])"; done
