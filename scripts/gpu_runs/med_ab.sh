python -m pytest tests/test_gpu_stein.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
python scripts/cfg1_plan.py 5
FCB_LIB_PATH=build_variants/agg1/libflowcover_b200.so python scripts/cfg1_plan.py 5
for v in "" build_variants/agg1/libflowcover_b200.so; do
FCB_LIB_PATH=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:median --log-file gpurun_out/cfg1_med_${v:+agg}.csv python scripts/cfg1_plan.py 1 > /dev/null 2>&1
done
