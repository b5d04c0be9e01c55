cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchlaw.py -q -k "tc_projection or cfg1_codes or benchlaw_codes or routed or counted or streamed" > gpurun_out/t_tcp.log 2>&1
echo "rc=$?" >> gpurun_out/t_tcp.log
PROBE_DEBUG=1 GEEK_PJ_TIMELINE=1 timeout 300 python tools/profile_step.py 2e7 > gpurun_out/tl0.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"project" --csv python tools/profile_step.py 2e7 > gpurun_out/tcp_launch.csv 2>&1
