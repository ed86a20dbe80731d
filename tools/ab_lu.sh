cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_lu_gpu.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/lu_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --only lu_f64_2048 > gpurun_out/lu_la.json 2>gpurun_out/lu_la.err
if [ -n "$ALT" ]; then
FB_LIB=$ALT timeout 600 python -m pytest tests/test_lu_gpu.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/lu_tests_alt.log
FB_LIB=$ALT timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --only lu_f64_2048 > gpurun_out/lu_alt.json 2>&1
fi
