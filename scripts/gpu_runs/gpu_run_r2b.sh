set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q -p no:cacheprovider > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/b_pytest.log
timeout 900 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo "bench rc=$?"
cat gpurun_out/b_bench.json; tail -20 gpurun_out/b_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; echo "ref rc=$?"
cat gpurun_out/b_ref.json; tail -5 gpurun_out/b_ref.err
