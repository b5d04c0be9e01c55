cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_project_kernel" -c 1 -o gpurun_out/tcp_final python tools/profile_step.py 1e8 > gpurun_out/tcp_final.log 2>&1
