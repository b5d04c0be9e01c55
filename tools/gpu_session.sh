cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rank_split" > gpurun_out/t_rs.log 2>&1
echo "rc=$?" >> gpurun_out/t_rs.log
