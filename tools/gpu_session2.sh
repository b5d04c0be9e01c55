cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -s > gpurun_out/t_multi.log 2>&1
echo "multi rc=$?" >> gpurun_out/t_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err
