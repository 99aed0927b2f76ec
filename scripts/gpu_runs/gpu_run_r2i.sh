set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/i_pytest.log
timeout 300 python scripts/configs.py 4 3 4s 1 2>/dev/null
timeout 900 python bench.py > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; echo "bench rc=$?"; cat gpurun_out/i_bench.json
