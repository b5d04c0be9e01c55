cd $GRAFT_REPO_ROOT
export PROBE_SORTED=1 PROBE_SCREENS=16,17 PROBE_MODES=0
for sl in 0 1 2; do GEEK_SCREEN_SLEEP=$sl timeout 600 python tools/screen_probe.py 20000000 963 128 >> gpurun_out/probe2.log 2>&1; done
