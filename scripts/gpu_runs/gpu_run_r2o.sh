set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/o_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/o_pytest.log
timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/o_bench.json 2> gpurun_out/o_bench.err; echo "bench rc=$?"; cat gpurun_out/o_bench.json
timeout 600 python scripts/configs.py 5 1 2>/dev/null
