cd $GRAFT_REPO_ROOT
timeout 600 python tools/profile_step.py 1e8 > gpurun_out/pstep.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"v2_|lex|radix|scan" --csv --log-file gpurun_out/v2_launches.csv python tools/profile_step.py 1e8 > gpurun_out/ncu_v2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_v2.log
