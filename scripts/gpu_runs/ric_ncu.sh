ncu --set full --clock-control none --import-source on -k regex:"ric_k2|plan_ric_k1" -c 2 -o gpurun_out/ric_full python scripts/lqr_time.py aircraft_3d 100000 1 > gpurun_out/ric_ncu.log 2>&1
tail -3 gpurun_out/ric_ncu.log
