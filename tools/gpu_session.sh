cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "singleton or table_by_table or mixed or sparse" > gpurun_out/t_single.log 2>&1
echo "rc=$?" >> gpurun_out/t_single.log
timeout 600 python tools/mixed_probe.py 20000000 > gpurun_out/mixed20m.log 2> gpurun_out/mixed20m.err
timeout 600 python tools/mixed_probe.py 50000000 > gpurun_out/mixed50m.log 2> gpurun_out/mixed50m.err
