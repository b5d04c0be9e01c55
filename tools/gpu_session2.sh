cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/multi2.log 2>&1
echo "rc=$?" >> gpurun_out/multi2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --no-checks > gpurun_out/bench2.json 2> gpurun_out/bench2.err
