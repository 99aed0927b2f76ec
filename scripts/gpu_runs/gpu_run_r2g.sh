set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for v in main r4m1 r4m2 r3m2; do
  if [ $v = main ]; then unset FCB_LIB_PATH; else export FCB_LIB_PATH=$PWD/build_variants/$v/libflowcover_b200.so; fi
  echo "== variant $v"
  timeout 300 python scripts/flow_cfg4.py 3
  timeout 300 python scripts/configs.py 4 3 2>/dev/null
done
unset FCB_LIB_PATH
