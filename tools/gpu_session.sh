cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "categorical or mixed or sparse" > gpurun_out/t_cat.log 2>&1
echo "rc=$?" >> gpurun_out/t_cat.log
timeout 300 python tools/cat_probe.py 50000000 39 13753 2000000 > gpurun_out/cat_probe.json 2> gpurun_out/cat_probe.err
timeout 300 python tools/cat_probe.py 20000000 13 4000 2000000 >> gpurun_out/cat_probe.json 2>> gpurun_out/cat_probe.err
timeout 600 python tools/mixed_probe.py 50000000 > gpurun_out/mixed50m.log 2> gpurun_out/mixed50m.err
