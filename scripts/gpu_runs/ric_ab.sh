set -x
python -m pytest tests/test_gpu_dynamics_lqr.py tests/test_gpu_plan.py tests/test_gpu_fused.py -x -q -m gpu 2>&1 | tail -3
for m in aircraft_3d diff_drive single_integrator_2d; do
  python scripts/lqr_time.py $m 100000 20
  FCB_LIB_PATH=scripts/lib_ric_old.so python scripts/lqr_time.py $m 100000 20
done
python scripts/lqr_time.py aircraft_3d 10000 50
FCB_LIB_PATH=scripts/lib_ric_old.so python scripts/lqr_time.py aircraft_3d 10000 50
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ric --csv python scripts/lqr_time.py aircraft_3d 100000 2 > gpurun_out/ric_new.csv 2>&1
FCB_LIB_PATH=scripts/lib_ric_old.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ric --csv python scripts/lqr_time.py aircraft_3d 100000 2 > gpurun_out/ric_old.csv 2>&1
