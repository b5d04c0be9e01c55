cd $GRAFT_REPO_ROOT
timeout 900 python tools/gist_probe.py 10000000 10000 > gpurun_out/gist.log 2>&1
echo "rc=$?" >> gpurun_out/gist.log
GEEK_NO_WIDE_GEMM=1 timeout 900 python tools/gist_probe.py 10000000 10000 > gpurun_out/gist_old.log 2>&1
