set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 300 python scripts/configs.py 4 3 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/h_pytest.log
timeout 900 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench rc=$?"; cat gpurun_out/h_bench.json
