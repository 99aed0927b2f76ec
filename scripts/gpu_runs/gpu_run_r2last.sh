set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/l_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/l_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/l_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/l_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/l_ref.json 2> gpurun_out/l_ref.err; echo "ref rc=$?"
