set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_tsp.py tests/test_gpu_guards.py -q -p no:cacheprovider > gpurun_out/k_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/k_pytest.log
timeout 900 python scripts/tsp_gpu_time.py 148 > gpurun_out/k_tsp_gpu.json; echo "tsp rc=$?"; cat gpurun_out/k_tsp_gpu.json
