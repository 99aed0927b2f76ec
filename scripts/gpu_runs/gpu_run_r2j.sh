set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/j_pytest.log
nproc
timeout 900 python scripts/tsp_baseline_time.py 32 16 "B200 box host" > gpurun_out/j_tsp.log 2>&1; echo "tsp rc=$?"; tail -2 gpurun_out/j_tsp.log
cp profiles/r02/tsp_baseline_cfg5_gpubox.json gpurun_out/ 2>/dev/null
