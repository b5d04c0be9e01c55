cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
