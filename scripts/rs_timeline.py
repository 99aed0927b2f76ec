"""Phase timeline of the resident flow kernel (FCB_TIMELINE builds of
flow_resident.cu; CTA 0 thread 0 marks).  Mean duration of every observed
(tag -> next tag) transition over a short config-2 plan.

    FCB_LIB_PATH=build_variants/rstl/libflowcover_b200.so python scripts/rs_timeline.py [iters] [T] [M]
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

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 12
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
M = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000
q = fc.benchmark_mixture(2)
Y = q.sample(M, [0, 2])
cfg = fc.PlanConfig(method="sinkhorn", eta=0.15 * T, max_iterations=iters, convergence_tol=0.0,
                    metric_interval=0)
lib = _lib.load()
lib.fcb_debug_rs_timeline.restype = ctypes.c_int
buf = (ctypes.c_ulonglong * 16384)()
disc = fc.Discretization(0.05, T, np.array([0.1, 0.1, 0.0, 0.0]))
fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y), disc, cfg)
lib.fcb_debug_rs_timeline(buf, 16384)  # reset
run = fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y), disc, cfg)
torch.cuda.synchronize()
k = lib.fcb_debug_rs_timeline(buf, 16384)
raw = np.array(buf[:k], dtype=np.uint64)
tags = (raw & np.uint64(0xFF)).astype(int)
t = (raw >> np.uint64(8)).astype(np.float64) / 1e3
stat = collections.defaultdict(list)
for i in range(len(tags) - 1):
    if tags[i] == 15:
        continue
    stat[(tags[i], tags[i + 1])].append(t[i + 1] - t[i])
names = {0: "start", 1: "setup", 2: "sync0", 3: "sweepA", 4: "sync1", 5: "reloadY", 6: "sweepB",
         7: "errred", 8: "sync2", 10: "compute", 11: "combine", 12: "self", 13: "syncS",
         14: "selfdone", 15: "end", 20: "A.init", 21: "A.loop", 22: "A.comb", 30: "B.init",
         31: "B.loop", 32: "B.comb", 40: "S.init", 41: "S.loop", 42: "S.comb"}
for key in sorted(stat, key=lambda k: -sum(stat[k])):
    v = stat[key]
    print(f"{names.get(key[0], key[0]):>9} -> {names.get(key[1], key[1]):<9} n={len(v):5d} "
          f"mean {np.mean(v):7.2f} us  total {np.sum(v):9.1f} us")
gaps = [t[i + 1] - t[i] for i in range(len(tags) - 1) if tags[i] == 15 and tags[i + 1] == 0]
if gaps:
    print(f"between flow launches (CTA 0 end -> next start): mean {np.mean(gaps):.1f} us, "
          f"median {np.median(gaps):.1f} us, n={len(gaps)}")
ka = run.flow_log[:, 1].sum()
ks = run.flow_log[:, 2].sum()
print(f"inner iterations: asym {ka:.0f} self {ks:.0f}; flows {len(run.flow_log)}")
