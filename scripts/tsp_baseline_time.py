"""Time the reference's TSP-waypoint baseline (tsp.py:276-316) on BASELINE
config-5 problems (single_integrator_2d, T=1000, problem b: seed b), on this
host's cores, with the UNMODIFIED reference imported read-only.  Build
container only (the reference is not on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 python scripts/tsp_baseline_time.py [problems]

Writes profiles/r02/tsp_baseline_cfg5.json (per-problem seconds, phase split,
extrapolation to 4096 problems on all cores, one problem per core).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import flowcover as fc  # noqa: E402
from flowcover.tsp import BaselineConfig, baseline_plan  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
model = fc.single_integrator_2d()
q = fc.benchmark_mixture(2)
rows = []
for b in range(k):
    t0 = time.perf_counter()
    res = baseline_plan(model, q, fc.Discretization(0.05, 1000, np.array([0.1, 0.1])),
                        BaselineConfig(seed=b))
    dt = time.perf_counter() - t0
    pt = res.phase_times
    rows.append({"problem": b, "seconds": dt, "tour_s": pt.flow, "lqr_s": pt.lqr,
                 "rollout_s": pt.rollout, "tour_length": float(res.tour.length)})
    print(rows[-1], flush=True)
cores = os.cpu_count() or 1
per = float(np.mean([r["seconds"] for r in rows]))
out = {"what": "reference tsp.baseline_plan, BASELINE config 5 problems (single_integrator_2d, "
               "T=1000, seed b), one process, FLOWCOVER_WORKERS unset",
       "host_cores": cores, "problems_timed": k, "mean_seconds_per_problem": per,
       "extrapolated_4096_problems_seconds_all_cores": per * 4096 / cores,
       "extrapolated": True, "rows": rows}
os.makedirs(os.path.join(ROOT, "profiles", "r02"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "r02", "tsp_baseline_cfg5.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps({k2: v for k2, v in out.items() if k2 != "rows"}))
