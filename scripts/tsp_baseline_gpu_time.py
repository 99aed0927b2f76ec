"""Time the whole TSP-waypoint baseline (targets, tour, resampling, 10 rounds of
TV-LQR tracking) on the GPU at config-5 shape: single_integrator_2d, T = 1000,
problem b with seed b -- the GPU counterpart of scripts/tsp_baseline_time.py
(the reference's baseline_plan on host cores).

    python scripts/tsp_baseline_gpu_time.py [problems]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m = fc.single_integrator_2d()
q = fc.benchmark_mixture(2)
disc = fc.Discretization(0.05, 1000, np.array([0.1, 0.1]))
fc.baseline_plan(m, q, disc, fc.BaselineConfig(seed=0))  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
res = [fc.baseline_plan(m, q, disc, fc.BaselineConfig(seed=b)) for b in range(B)]
dt = time.perf_counter() - t0
pt = [r.phase_times for r in res]
print(json.dumps({
    "what": "GPU baseline_plan (tour + arc-length resampling + 10 TV-LQR tracking rounds), "
            "single_integrator_2d, T=1000, one problem per call",
    "problems": B, "seconds": dt, "seconds_per_problem": dt / B,
    "mean_phase_s": {"tour": float(np.mean([p.flow for p in pt])),
                     "lqr_device": float(np.mean([p.lqr for p in pt])),
                     "rollout_device": float(np.mean([p.rollout for p in pt]))},
    "projected_4096_problems_s": 4096 * dt / B}))
# batched: all tours in one launch (one CTA per problem), then the tracking
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 512
cfgs = [fc.BaselineConfig(seed=b) for b in range(NB)]
torch.cuda.synchronize()
t0 = time.perf_counter()
res = fc.baseline_plans(m, q, disc, cfgs)
dt = time.perf_counter() - t0
print(json.dumps({
    "what": "GPU baseline_plans (batched tours + per-problem tracking), same problems",
    "problems": NB, "seconds": dt, "seconds_per_problem": dt / NB,
    "projected_4096_problems_s": 4096 * dt / NB}))
