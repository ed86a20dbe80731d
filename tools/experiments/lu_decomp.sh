cd $GRAFT_REPO_ROOT
rm -f gpurun_out/lu_decomp.txt
for d in 0 3 4; do
for g in 1 0; do
FB_LU_GRAPH=$g FB_LU_DEBUG=$d timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --only lu_f64_2048 > gpurun_out/lu_d.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/lu_d.json').read().strip().splitlines()[-1]); print('debug', $d, 'graph', $g, d['blocks']['lu_f64_2048']['ms_per_step'])" >> gpurun_out/lu_decomp.txt
done
done
