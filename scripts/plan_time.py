"""Time config-2 plans (device events) with the fused planner on/off."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
q = fc.benchmark_mixture(2)
Y = q.sample(10_000, [0, 2])
cfg = fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=iters, convergence_tol=0.0,
                    metric_interval=0)
disc = fc.Discretization(0.05, 2000, np.array([0.1, 0.1, 0.0, 0.0]))
for mode in ("1", "0", "1"):
    os.environ["FCB_FUSED"] = mode
    run = fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y), disc, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run = fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y), disc, cfg)
    e1.record()
    torch.cuda.synchronize()
    r = run.result
    print(f"fused={mode}: {e0.elapsed_time(e1):.2f} ms, iters {r.iterations_used}, "
          f"pairs {run.pairs:.4e}, phases {r.phase_times}, S[-1] {r.trajectory.S[-1]}, "
          f"flow_norm[-1] {r.flow_norms[-1]:.6e} cost[-1] {r.lqr_costs[-1]:.6e}")
