set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo "bench rc=$?"; cat gpurun_out/e_bench.json
timeout 600 python scripts/configs.py 1 5 5full > gpurun_out/e_cfg.jsonl 2> gpurun_out/e_cfg.err; echo "cfg rc=$?"; cat gpurun_out/e_cfg.jsonl; tail -3 gpurun_out/e_cfg.err
timeout 300 python scripts/flow_cfg4.py 3
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_driver.py > gpurun_out/e_san_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/e_san_$tool.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flow_kernel -c 1 --launch-skip 1 -o gpurun_out/e_flow_cfg4 python scripts/flow_cfg4.py 2 > gpurun_out/e_ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/e_ncu_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/e_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-secondary > gpurun_out/e_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
