# Round-2 additions to tools/profile_round.sh: ncu --set full of the kernels added late in the
# round (256^2 cluster kernel, the 16384^2 four-step column passes, the mixed-radix line kernel).
# Each ncu command follows the same command run without ncu (exit 0).
cd $GRAFT_REPO_ROOT
R=${R:-r2}
SCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --only fft2d_256_fwd_inv"
timeout 600 $SCMD > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft256_cluster" -s 4 -c 2 -o gpurun_out/${R}_fft256 $SCMD > gpurun_out/${R}_fft256.log 2>&1
CCMD="python tools/fft_pass_bench.py 16384 16384 1"
timeout 600 $CCMD > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_pass_tma" -s 2 -c 2 -o gpurun_out/${R}_fft16k_cols $CCMD > gpurun_out/${R}_fft16k_cols.log 2>&1
MCMD="python tools/fft_pass_bench.py 1000 1000 5"
timeout 600 $MCMD > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mr_lines|bs_transpose" -s 6 -c 3 -o gpurun_out/${R}_mixed $MCMD > gpurun_out/${R}_mixed.log 2>&1
ls gpurun_out/*.ncu-rep
