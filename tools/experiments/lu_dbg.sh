cd $GRAFT_REPO_ROOT
python tools/lu_dbg.py > gpurun_out/lu_dbg.txt 2>&1
bash tools/ab_lu.sh
