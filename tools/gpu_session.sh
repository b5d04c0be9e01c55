cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests/test_gpu_benchlaw.py tests/test_gpu_transport.py "tests/test_gpu_parity.py::test_rank_split_random_vs_oracle" -x -q > gpurun_out/t_new.log 2>&1
echo "new rc=$?" >> gpurun_out/t_new.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/t_all.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
