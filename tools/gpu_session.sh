cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -x -m gpu > gpurun_out/t_all.log 2>&1
echo "rc=$?" >> gpurun_out/t_all.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_skip.json 2> gpurun_out/bench_skip.err
