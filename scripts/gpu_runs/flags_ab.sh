# per-slice publication flags (default) vs the two grid barriers (RS_FLAGS=0) on config 2
python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity_r2.py tests/test_gpu_sinkhorn.py tests/test_gpu_plan.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
for r in 1 2 3; do
  for v in "" build_variants/noflags/libflowcover_b200.so; do
    echo "${v:-flags}: $(FCB_LIB_PATH=$v python scripts/plan_time.py 200 2>/dev/null | grep 'fused=1' | tail -1 | cut -d, -f1,4)"
  done
done
