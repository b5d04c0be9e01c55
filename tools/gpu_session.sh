cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-checks --no-e2e > gpurun_out/bench3.json 2> gpurun_out/bench3.err
