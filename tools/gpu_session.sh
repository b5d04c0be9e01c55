cd $GRAFT_REPO_ROOT
timeout 1200 python tools/sparse_probe.py 20000000 > gpurun_out/sparse_now.json 2> gpurun_out/sparse_now.err
