# A/B: Riccati K1 walk / K3 step in Riccati form (default) vs the generic combines
V=build_variants/ricgen/libflowcover_b200.so
python -m pytest tests/test_gpu_dynamics_lqr.py tests/test_gpu_plan.py tests/test_gpu_fused.py tests/test_gpu_parity_r2.py tests/test_gpu_distributed.py tests/test_gpu_tsp.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
for m in aircraft_3d diff_drive; do
  python scripts/lqr_time.py $m 100000 20
  FCB_LIB_PATH=$V python scripts/lqr_time.py $m 100000 20
done
python scripts/lqr_time.py diff_drive 10000 50
FCB_LIB_PATH=$V python scripts/lqr_time.py diff_drive 10000 50
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ric --csv python scripts/lqr_time.py aircraft_3d 100000 2 > gpurun_out/ric2_new.csv 2>&1
