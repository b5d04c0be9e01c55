cd $GRAFT_REPO_ROOT
timeout 600 python tools/profile_step.py 1e8 > gpurun_out/pstep.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tc_screen_kernel|emit_winners|tc_classify2|tc_recheck8" -c 4 -o gpurun_out/r2_screen python tools/profile_step.py 1e8 > gpurun_out/ncu_screen.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_screen.log
