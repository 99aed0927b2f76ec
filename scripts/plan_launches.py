"""A short config-2 plan for launch-list profiling (ncu --metrics gpu__time_duration.sum)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 6
q = fc.benchmark_mixture(2)
Y = q.sample(10_000, [0, 2])
cfg = fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=iters, convergence_tol=0.0,
                    metric_interval=0)
disc = fc.Discretization(0.05, 2000, np.array([0.1, 0.1, 0.0, 0.0]))
fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y), disc, cfg)
