set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flow_kernel -c 1 --launch-skip 1 -o gpurun_out/q_flow_cfg4 python scripts/flow_cfg4.py 2 > gpurun_out/q_ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_lines.py gpurun_out/q_flow_cfg4.ncu-rep > gpurun_out/q_lines.txt 2>&1
timeout 900 python scripts/shard_projection.py 1 2 4 8 > gpurun_out/q_proj.jsonl 2> gpurun_out/q_proj.err; echo "proj rc=$?"; tail -1 gpurun_out/q_proj.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/q_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-secondary > gpurun_out/q_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
