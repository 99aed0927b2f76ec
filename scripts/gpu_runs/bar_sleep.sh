# grid-barrier poll interval A/B on the config-2 fused planner (3 alternating rounds)
for r in 1 2 3; do
  for v in "" build_variants/bs0/libflowcover_b200.so build_variants/bs100/libflowcover_b200.so; do
    echo "${v:-default(20ns)}: $(FCB_LIB_PATH=$v python scripts/plan_time.py 200 2>/dev/null | grep 'fused=1' | tail -1 | cut -d, -f1)"
  done
done
