cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchlaw.py -q -x > gpurun_out/t_all.log 2>&1
echo "rc=$?" >> gpurun_out/t_all.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_bnd.json 2> gpurun_out/bench_bnd.err
