python scripts/cfg1_plan.py 5
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg1_launches.csv python scripts/cfg1_plan.py 1 > /dev/null 2>&1
echo ncu rc=$?
