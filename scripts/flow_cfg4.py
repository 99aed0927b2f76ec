"""Config-4 Sinkhorn flows (aircraft_3d, T=1e5, M=1e6) on one GPU, for ncu.

    python scripts/flow_cfg4.py [reps]

X = workspace projection of the initial rollout (random-small controls,
stream [0, 1]); Y = benchmark_mixture(3) draws (stream [0, 2]).  Prints the
per-flow time and the executed pairs.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m = fc.aircraft_3d()
T, M = 100_000, 1_000_000
cfg = fc.PlanConfig(method="sinkhorn", seed=0)
U0 = fc.initial_controls(cfg, m, T)
S = fc.rollout(m, fc.default_start(m), U0, 0.05)
X = m.project_states(S[1:])
Y = fc.benchmark_mixture(3).sample(M, [0, 2])
q = fc.SamplePoints(Y)
for i in range(reps):
    st = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fc.sinkhorn_flow(X, q, fc.SinkhornConfig(), stats=st)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    pairs = 2.0 * st["iters_cross"] * T * M + st["iters_self"] * T * T
    print(f"flow {i}: {dt * 1e3:.1f} ms (incl. host copies), inner {st['iters_cross']}/"
          f"{st['iters_self']}, {pairs:.3e} pairs, {pairs / dt:.3e} pair/s", flush=True)
