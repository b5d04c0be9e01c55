cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/final_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
