set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/m_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/m_pytest.log
/usr/bin/time -v timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; echo "bench rc=$?"; cat gpurun_out/m_bench.json; grep "Elapsed" gpurun_out/m_bench.err
/usr/bin/time -v timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err; echo "ref rc=$?"; cat gpurun_out/m_ref.json; grep "Elapsed" gpurun_out/m_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/m_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-secondary > gpurun_out/m_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
