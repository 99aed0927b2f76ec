"""Phase timeline of the fused planner (FCB_TIMELINE build, CTA 0 stamps).

    FCB_LIB_PATH=build_variants/pltl/libflowcover_b200.so python scripts/plan_timeline.py [iters]
"""
import collections
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _lib  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
q = fc.benchmark_mixture(2)
Y = q.sample(10_000, [0, 2])
cfg = fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=iters, convergence_tol=0.0,
                    metric_interval=0)
disc = fc.Discretization(0.05, 2000, np.array([0.1, 0.1, 0.0, 0.0]))
lib = _lib.load()
buf = (ctypes.c_ulonglong * 16384)()
fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y), disc, cfg)
lib.fcb_debug_plan_timeline(buf, 16384)
fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y), disc, cfg)
torch.cuda.synchronize()
k = lib.fcb_debug_plan_timeline(buf, 16384)
raw = np.array(buf[:max(k, 0)], dtype=np.uint64)
tags = (raw & np.uint64(0xFF)).astype(int)
t = (raw >> np.uint64(8)).astype(np.float64) / 1e3
names = {50: "it", 51: "roll.p1", 52: "roll.sync1", 53: "roll.p2", 54: "roll.sync2", 55: "roll.chk",
         56: "flow", 57: "eta.p1", 58: "eta.sync", 59: "eta.p2+z.p1", 60: "z.sync", 61: "z.p2"}
stat = collections.defaultdict(list)
for i in range(len(tags) - 1):
    a, b = tags[i], tags[i + 1]
    if a in names and b in names:
        stat[(a, b)].append(t[i + 1] - t[i])
for key in sorted(stat, key=lambda k: -sum(stat[k])):
    v = stat[key]
    print(f"{names[key[0]]:>12} -> {names[key[1]]:<12} n={len(v):4d} mean {np.mean(v):7.2f} us")
