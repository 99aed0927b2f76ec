# A/B of the FMA-pipe exp2 (FCB_EMU_EX2) on the config-4 flows and the bench
V=build_variants/emu1/libflowcover_b200.so
python scripts/flow_cfg4.py 3
FCB_LIB_PATH=$V python scripts/flow_cfg4.py 3
FCB_LIB_PATH=$V python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_sinkhorn.py -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 3 --warmup 3 > gpurun_out/emu0_bench.json 2>gpurun_out/emu0_bench.err
FCB_LIB_PATH=$V python bench.py --steps 3 --warmup 3 > gpurun_out/emu1_bench.json 2>gpurun_out/emu1_bench.err
python - <<'PY'
import json
for n in ("emu0","emu1"):
    d=json.load(open(f"gpurun_out/{n}_bench.json"))
    r=d["roofline"]
    print(n, d["value"], d["ms_per_step"], r["frac"], r.get("sinkhorn_flow_Gpair_s"), d["clocks"])
PY
