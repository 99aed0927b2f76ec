set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/f_pytest.log
timeout 300 python scripts/flow_cfg4.py 3
timeout 900 python bench.py --no-cpu > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"; cat gpurun_out/f_bench.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flow_kernel -c 1 --launch-skip 1 -o gpurun_out/f_flow_cfg4 python scripts/flow_cfg4.py 2 > gpurun_out/f_ncu_full.log 2>&1; echo "ncu full rc=$?"
