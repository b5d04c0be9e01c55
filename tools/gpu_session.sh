cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -x -m gpu > gpurun_out/t_all.log 2>&1
echo "rc=$?" >> gpurun_out/t_all.log
