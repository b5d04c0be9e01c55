cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "screen or assign or tcgen05 or bound" > gpurun_out/t_scr.log 2>&1
echo "rc=$?" >> gpurun_out/t_scr.log
export PROBE_DEBUG=1 PROBE_SORTED=1
PROBE_MODES=0,1 timeout 600 python tools/screen_probe.py 20000000 963 128 >> gpurun_out/scr_dbg11.log 2>&1
PROBE_MODES=0 timeout 600 python tools/screen_probe.py 20000000 1000 128 >> gpurun_out/scr_dbg11.log 2>&1
