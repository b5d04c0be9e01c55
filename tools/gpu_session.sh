cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchlaw.py -q -x -k "seeding or vote or pipeline or benchlaw or silk or winners" > gpurun_out/t_vote.log 2>&1
echo "rc=$?" >> gpurun_out/t_vote.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-checks --no-e2e > gpurun_out/bench5.json 2> gpurun_out/bench5.err
