set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/w_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/w_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/w_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/w_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/w_bench.json 2> gpurun_out/w_bench.err; echo "bench rc=$?"
cat gpurun_out/w_bench.json | cut -c1-600
