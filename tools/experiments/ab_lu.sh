cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_lu_gpu.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/lu_tests.log
rm -f gpurun_out/lu_ab.txt
for cfg in "" "FB_LU_GRAPH=0"; do
env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --only lu_f64_2048 > gpurun_out/lu_x.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/lu_x.json').read().strip().splitlines()[-1]); print('$cfg', d['blocks']['lu_f64_2048']['ms_per_step'])" >> gpurun_out/lu_ab.txt
done
