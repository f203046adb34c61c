cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:ccl_runs -s 1 -c 1 -o gpurun_out/ccl_runs_16384 python tools/profile_ccl.py 16384 100 > gpurun_out/ccl_prof.log 2>&1
