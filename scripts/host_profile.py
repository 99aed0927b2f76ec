"""Host-side profile of the config-4 bench step (cProfile over plan_detailed).

    python scripts/host_profile.py
"""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _dev  # noqa: E402

model = fc.aircraft_3d()
Y = bench.targets4()
q3 = fc.benchmark_mixture(3)
disc = fc.Discretization(bench.DT, bench.T4, fc.default_start(model))
cfg_sk = fc.PlanConfig(method="sinkhorn", eta=bench.ETA_SK, max_iterations=3, convergence_tol=0.0,
                       metric_interval=0, seed=0)
cfg_sv = fc.PlanConfig(method="stein", eta=bench.ETA_SV, max_iterations=3, convergence_tol=0.0,
                       metric_interval=0, seed=0, stein=fc.SteinConfig(bandwidth=bench.H_SV))
Yd = _dev.f64(Y)


def step():
    fc.plan_detailed(model, fc.SamplePoints(Y), disc, cfg_sk, resident_targets=Yd)
    fc.plan_detailed(model, q3, disc, cfg_sv)


for _ in range(2):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
