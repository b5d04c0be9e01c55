cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/ -q -x -m gpu > gpurun_out/t_all.log 2>&1
echo "rc=$?" >> gpurun_out/t_all.log
GEEK_SPLIT_CSHIFT=4 GEEK_PROFILE=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-checks --no-e2e > gpurun_out/bc_4.json 2> gpurun_out/bc_4.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_gc.json 2> gpurun_out/bench_gc.err
