# config-5 (batched CTA-group planner) layout A/B via the FCB_RS_PLAN_* overrides
for v in X=0 FCB_RS_PLAN_A=4,6 FCB_RS_PLAN_A=3,4 FCB_RS_PLAN_A=5,6 FCB_RS_PLAN_A=4,4 FCB_RS_PLAN_B=4,4 FCB_RS_PLAN_B=3,3 FCB_RS_PLAN_B=5,4 FCB_RS_PLAN_B=5,2 FCB_RS_PLAN_S=4,4 FCB_RS_PLAN_S=5,4 X=1; do
  echo "== $v $(env $v python scripts/configs.py 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['seconds'],4), round(d['frac_of_mufu'],4))")"
done
