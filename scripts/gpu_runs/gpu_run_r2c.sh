set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
python scripts/debug/shard_merge.py
python scripts/lqr_time.py aircraft_3d 100000 10
python scripts/lqr_time.py diff_drive 10000 10
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/c_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/c_pytest.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_lqr_launches.csv python scripts/lqr_time.py aircraft_3d 100000 2 > /dev/null 2>&1
