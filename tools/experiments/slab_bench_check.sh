cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --slab --steps 4 --warmup 3 > gpurun_out/slab1.json 2> gpurun_out/slab1.err
FB_SLAB_FUSED=0 timeout 600 python bench.py --slab --steps 4 --warmup 3 > gpurun_out/slab1_nccl.json 2>> gpurun_out/slab1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --slab --steps 4 --warmup 3 > gpurun_out/slab_trun.json 2>> gpurun_out/slab1.err
