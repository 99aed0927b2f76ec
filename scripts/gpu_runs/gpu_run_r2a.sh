set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python scripts/configs.py 4 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"
cat gpurun_out/cfg4.jsonl; tail -5 gpurun_out/cfg4.err
