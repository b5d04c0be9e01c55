cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/final_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 3 --no-checks --no-e2e > gpurun_out/final_ncu.log 2>&1
