cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/smi4.txt
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -s > gpurun_out/t_multi4.log 2>&1
echo "multi rc=$?" >> gpurun_out/t_multi4.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_g$N.json 2> gpurun_out/bench_g$N.err
done
