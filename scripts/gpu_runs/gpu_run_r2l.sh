set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flow_kernel -c 1 --launch-skip 1 -o gpurun_out/l_flow_cfg4 python scripts/flow_cfg4.py 2 > gpurun_out/l_ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_lines.py gpurun_out/l_flow_cfg4.ncu-rep > gpurun_out/l_lines.txt 2>&1; head -50 gpurun_out/l_lines.txt
