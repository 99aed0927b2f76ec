set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/p_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/p_pytest.log
timeout 900 python bench.py --no-cpu --steps 10 > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; echo "bench rc=$?"; python -c "import json; b=json.load(open('gpurun_out/p_bench.json')); print(b['value'], b['ms_per_step'], b['roofline']['frac'], b['secondary'])"
timeout 600 python scripts/configs.py 5 2>/dev/null
