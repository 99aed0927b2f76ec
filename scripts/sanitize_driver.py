"""One small call of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python scripts/sanitize_driver.py
    compute-sanitizer --tool racecheck python scripts/sanitize_driver.py
    compute-sanitizer --tool synccheck python scripts/sanitize_driver.py

Shapes are small (the tools replay / instrument every access), but each one is
chosen to take the code path the BASELINE configs take: the shared-memory
resident flow and the persistent planner (grid-group barriers), the chunked
cooperative solver (GridBarrier), the sharded steps, the radix median, the
warp-cooperative Riccati scan and the affine scans (one-launch and chunked).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import distributed as D  # noqa: E402

rng = np.random.default_rng(0)
q2, q3 = fc.benchmark_mixture(2), fc.benchmark_mixture(3)
only = set(sys.argv[1:])


def step(name):
    return not only or name in only


if step("flows"):
    X, Y = q2.sample(700, [1, 2]), q2.sample(1500, [0, 2])
    fc.sinkhorn_flow(X, fc.SamplePoints(Y), fc.SinkhornConfig(precision="float32"))  # resident
    os.environ["FCB_RESIDENT"] = "0"
    fc.sinkhorn_flow(X, fc.SamplePoints(Y), fc.SinkhornConfig(precision="float32"))  # chunked
    fc.sinkhorn_flow(X, fc.SamplePoints(Y), fc.SinkhornConfig(precision="float64"))
    os.environ["FCB_RESIDENT"] = "1"
    X3, Y3 = q3.sample(300, [1, 3]), q3.sample(900, [0, 2])
    fc.sinkhorn_flow(X3, fc.SamplePoints(Y3), fc.SinkhornConfig(precision="float32"))
    fc.entropic_ot(X, Y, fc.SinkhornConfig())
    fc.sinkhorn_divergence(X, Y, fc.SinkhornConfig())
    print("flows ok", flush=True)

if step("stein"):
    P = q2.sample(600, [3, 2])
    fc.stein_flow(P, q2, fc.SteinConfig(precision="float32"))
    fc.stein_flow(q3.sample(500, [3, 3]), q3, fc.SteinConfig(bandwidth=0.02))
    print("stein ok", flush=True)

if step("dyn"):
    for name, T in (("single_integrator_2d", 300), ("diff_drive", 300), ("aircraft_3d", 300),
                    ("aircraft_3d", 20_000)):
        m = fc.get_model(name)
        U = 1e-2 * rng.standard_normal((T, m.control_dim))
        S = fc.rollout(m, fc.default_start(m), U, 0.05)
        ltv = fc.linearize_along(m, S, U, 0.05)
        w = fc.workspace_weights(m.project_matrix, m.control_dim)
        a = 1e-3 * rng.standard_normal((T, m.state_dim))
        fc.solve_flow_lqr(ltv, a, w)
    print("dynamics/lqr ok", flush=True)

if step("plans"):
    di = fc.double_integrator_2d()
    s0 = np.array([0.1, 0.1, 0.0, 0.0])
    tg = fc.SamplePoints(q2.sample(1200, [0, 2]))
    cfg = fc.PlanConfig(method="sinkhorn", eta=45.0, max_iterations=4, convergence_tol=0.0,
                        metric_interval=0, sinkhorn=fc.SinkhornConfig(precision="float32"))
    fc.plan(di, tg, fc.Discretization(0.05, 300, s0), cfg)  # fused persistent planner
    fc.plan(fc.aircraft_3d(), fc.SamplePoints(q3.sample(900, [0, 2])),
            fc.Discretization(0.05, 300, fc.default_start(fc.aircraft_3d())),
            fc.PlanConfig(method="sinkhorn", eta=30.0, max_iterations=3, convergence_tol=0.0,
                          metric_interval=2))
    fc.plan(di, q2, fc.Discretization(0.05, 200, s0),
            fc.PlanConfig(method="stein", eta=0.1, max_iterations=3, convergence_tol=0.0,
                          metric_interval=0))
    m = fc.single_integrator_2d()
    probs = [(m, fc.SamplePoints(q2.sample(512, [b, 2])), fc.Discretization(0.05, 256,
              np.array([0.1, 0.1])), fc.PlanConfig(method="sinkhorn", eta=30.0, max_iterations=3,
              convergence_tol=0.0, metric_interval=0, seed=b,
              sinkhorn=fc.SinkhornConfig(precision="float32"))) for b in range(4)]
    fc.plan_batch(probs)
    print("plans ok", flush=True)

if step("shard"):
    X, Y = q3.sample(400, [1, 3]), q3.sample(1300, [0, 2])
    D.ShardedSinkhornFlow(Y, fc.SinkhornConfig(precision="float32"))(X)
    sv = D.ShardedStein(400, 3, q3, 0.02)
    Xd = torch.from_numpy(X).cuda()
    out = torch.zeros((400, 3), dtype=torch.float64, device="cuda")
    sv.flow_into(Xd, out, torch.zeros(8, dtype=torch.float64, device="cuda"))
    print("shard ok", flush=True)

torch.cuda.synchronize()
print("sanitize driver done")
