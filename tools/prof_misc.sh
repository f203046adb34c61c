# ncu captures for DESIGN/profiles: CCL tile kernel (16384^2), planar 4096^2, cluster 400^2
cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:ccl_runs -s 1 -c 1 -f -o gpurun_out/r02b_ccl_runs_16384 python tools/profile_ccl.py 16384 100 > gpurun_out/prof_ccl.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:planar_pass -s 40 -c 1 -f -o gpurun_out/r02b_planar_4096 python tools/profile_pass.py 4096 4096 20 8 > gpurun_out/prof_4096.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:cluster_kernel -c 1 -f -o gpurun_out/r02b_cluster_400 python tools/profile_cluster.py 200 > gpurun_out/prof_cluster.log 2>&1
