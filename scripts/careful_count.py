"""Per-flow count of chunked-solver work items that fell back to the careful
loop, over a config-4 Sinkhorn plan (one GPU).

    python scripts/careful_count.py [iters]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _lib  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m = fc.aircraft_3d()
T, M = 100_000, 1_000_000
Y = fc.benchmark_mixture(3).sample(M, [0, 2])
lib = _lib.load()
cfg = fc.PlanConfig(method="sinkhorn", eta=15000.0, max_iterations=1, convergence_tol=0.0,
                    metric_interval=0, seed=0)
disc = fc.Discretization(0.05, T, fc.default_start(m))
lib.fcb_debug_careful_items()
run = fc.plan_detailed(m, fc.SamplePoints(Y), disc, fc.PlanConfig(**{**cfg.__dict__, "max_iterations": iters}))
torch.cuda.synchronize()
print("careful items over the plan:", lib.fcb_debug_careful_items(), "flow_log", run.flow_log.tolist(),
      "phase flow s", run.result.phase_times.flow)
# the same flows one by one on the plan's own states
S = run.result.trajectory.S
X = m.project_states(S[1:])
print("final X extent", np.ptp(X, axis=0))
