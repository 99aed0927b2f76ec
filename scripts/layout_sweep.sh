# Config-2 A/B timing of the resident flow's sweep thread layouts on one GPU:
#   bash scripts/layout_sweep.sh [VAR=cg_log,rows ...]   (results in gpurun_out/l_sweep.txt)
mkdir -p gpurun_out
run() { echo "== $1" >> gpurun_out/l_sweep.txt; env $1 timeout 200 python bench.py --no-cpu --steps 3 --warmup 3 2>>gpurun_out/l_sweep.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline']['frac'])" >> gpurun_out/l_sweep.txt 2>&1; }
if [ $# -eq 0 ]; then set -- X=0 FCB_RS_PLAN_B=9,4 FCB_RS_PLAN_B=8,4 FCB_RS_PLAN_B=6,2 FCB_RS_PLAN_B=5,1 \
    FCB_RS_PLAN_A=6,6 FCB_RS_PLAN_A=4,3 FCB_RS_PLAN_S=9,4 FCB_RS_PLAN_S=7,4; fi
for v in "$@"; do run "$v"; done
echo done >> gpurun_out/l_sweep.txt
