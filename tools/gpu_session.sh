cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchlaw.py -q -k "tc_projection or cfg1_codes or benchlaw_codes or routed or counted or streamed" > gpurun_out/t_tcp.log 2>&1
echo "rc=$?" >> gpurun_out/t_tcp.log
