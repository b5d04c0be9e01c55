cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -s > gpurun_out/t_multi.log 2>&1
echo "multi rc=$?" >> gpurun_out/t_multi.log
