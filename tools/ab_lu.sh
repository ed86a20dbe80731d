cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_lu_gpu.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/lu_tests.log
rm -f gpurun_out/lu_ab.txt
for cfg in "" "FB_LU_TMA=0" "FB_LU_DEBUG=3" "FB_LU_DEBUG=4"; do
env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --only lu_f64_2048 > gpurun_out/lu_x.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/lu_x.json').read().strip().splitlines()[-1]); print('$cfg', d['blocks']['lu_f64_2048']['ms_per_step'])" >> gpurun_out/lu_ab.txt
done
FB_LIB=paper_2004_09883_b200/libfb_lutime.so timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --only lu_f64_2048 2>&1 | grep LU_TIMING | head -3 > gpurun_out/lu_timing.txt
