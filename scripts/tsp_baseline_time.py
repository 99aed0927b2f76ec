"""Time the reference's TSP-waypoint baseline (tsp.py:276-316) on BASELINE
config-5 problems (single_integrator_2d, T=1000, problem b: seed b), on this
host's cores, with the UNMODIFIED reference imported read-only.  Build
container only (the reference is not on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 python scripts/tsp_baseline_time.py [problems] [processes] [label]

Writes profiles/r02/tsp_baseline_cfg5*.json (per-problem seconds, phase split,
throughput with one problem per process, extrapolation to 4096 problems).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the unmodified reference: read-only source tree here, or its pip install
# under baseline/_ref (which also travels to the GPU box)
_SRC = "/root/reference/pkg/src"
sys.path.insert(0, _SRC if os.path.isdir(_SRC) else os.path.join(ROOT, "baseline", "_ref"))
import flowcover as fc  # noqa: E402
from flowcover.tsp import BaselineConfig, baseline_plan  # noqa: E402


def one(b):
    model = fc.single_integrator_2d()
    q = fc.benchmark_mixture(2)
    t0 = time.perf_counter()
    res = baseline_plan(model, q, fc.Discretization(0.05, 1000, np.array([0.1, 0.1])),
                        BaselineConfig(seed=b))
    dt = time.perf_counter() - t0
    pt = res.phase_times
    return {"problem": b, "seconds": dt, "tour_s": pt.flow, "lqr_s": pt.lqr,
            "rollout_s": pt.rollout, "tour_length": float(res.tour.length)}


if __name__ == "__main__":
    import multiprocessing as mp

    k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    procs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    label = sys.argv[3] if len(sys.argv) > 3 else "build container"
    os.environ.setdefault("FLOWCOVER_WORKERS", "1")
    t0 = time.perf_counter()
    if procs > 1:
        with mp.get_context("spawn").Pool(procs) as pool:
            rows = pool.map(one, range(k))
    else:
        rows = [one(b) for b in range(k)]
    wall = time.perf_counter() - t0
    for r in rows:
        print(r, flush=True)
    cores = os.cpu_count() or 1
    per = float(np.mean([r["seconds"] for r in rows]))
    out = {"what": "reference tsp.baseline_plan, BASELINE config 5 problems (single_integrator_2d, "
                   "T=1000, problem b: seed b), one problem per process",
           "host": label, "host_cores": cores, "processes": procs, "problems_timed": k,
           "wall_seconds": wall, "mean_seconds_per_problem": per,
           "problems_per_second_all_processes": k / wall,
           "extrapolated_4096_problems_seconds": 4096 / (k / wall),
           "extrapolated": True, "rows": rows}
    os.makedirs(os.path.join(ROOT, "profiles", "r02"), exist_ok=True)
    name = "tsp_baseline_cfg5.json" if label == "build container" else "tsp_baseline_cfg5_gpubox.json"
    with open(os.path.join(ROOT, "profiles", "r02", name), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k2: v for k2, v in out.items() if k2 != "rows"}))
