"""BASELINE config 1 (double integrator, SVGD median h, T=500, 100 iterations), a few plans."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
di = fc.double_integrator_2d()
q = fc.benchmark_mixture(2)
disc = fc.Discretization(0.05, 500, np.array([0.1, 0.1, 0.0, 0.0]))
cfg = fc.PlanConfig(method="stein", eta=0.1, max_iterations=100, convergence_tol=0.0,
                    metric_interval=0)
fc.plan_detailed(di, q, disc, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    r = fc.plan_detailed(di, q, disc, cfg)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
pt = r.result.phase_times
print(f"config 1: {dt * 1e3:.2f} ms per plan, {100 / dt:.0f} it/s; phase (device) flow "
      f"{pt.flow * 1e3:.2f} lqr {pt.lqr * 1e3:.2f} rollout {pt.rollout * 1e3:.2f} ms")
