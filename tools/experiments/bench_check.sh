cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --only gemm_f32_32768 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/b32k.json 2> gpurun_out/b32k.err
timeout 900 python bench.py --slab --steps 3 --warmup 3 > gpurun_out/bslab.json 2>> gpurun_out/b32k.err
