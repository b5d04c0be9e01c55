cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -x -m gpu -k "seeding or bins or trace or mixed or sparse or worked or table_by_table" > gpurun_out/t_seed.log 2>&1
echo "rc=$?" >> gpurun_out/t_seed.log
timeout 900 python tools/mixed_probe.py 20000000 > gpurun_out/mixed20m.log 2>&1
timeout 1800 python tools/mixed_probe.py 50000000 > gpurun_out/mixed50m.log 2>&1
