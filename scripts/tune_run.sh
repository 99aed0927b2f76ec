#!/bin/bash
# Run the sweep/solve microbenchmarks for every build variant.
cd "$(dirname "$0")/.."
for d in build_variants/*/; do
  name=$(basename $d)
  for cap in ${CAPS:-2 3 4}; do
    echo "== $name cap=$cap"
    for s in "2000 10000" "10000 100000" "100000 1000000"; do
      FCB_LIB_PATH=$d/libflowcover_b200.so FCB_OT_CTAS_PER_SM=$cap timeout 120 python scripts/profile_ot.py sweep $s 2>&1 | tail -1
    done
    FCB_LIB_PATH=$d/libflowcover_b200.so FCB_OT_CTAS_PER_SM=$cap timeout 120 python scripts/profile_ot.py solve 2>&1 | tail -1
  done
done
