"""Barrier timeline of the one-launch flow kernel inside the planner
(FCB_TIMELINE builds; block 0's globaltimer at every grid-barrier arrival and
release).

    FCB_LIB_PATH=build_variants/tl/libflowcover_b200.so python scripts/flow_timeline.py [iters]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _lib  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 12
q = fc.benchmark_mixture(2)
Y = q.sample(10_000, [0, 2])
cfg = fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=iters, convergence_tol=0.0,
                    metric_interval=0)
lib = _lib.load()
buf = (ctypes.c_ulonglong * 8192)()
run = fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y),
                       fc.Discretization(0.05, 2000, np.array([0.1, 0.1, 0.0, 0.0])), cfg)
lib.fcb_debug_timeline(buf, 8192)  # reset
run = fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y),
                       fc.Discretization(0.05, 2000, np.array([0.1, 0.1, 0.0, 0.0])), cfg)
torch.cuda.synchronize()
k = lib.fcb_debug_timeline(buf, 8192)
t = np.array(buf[:k], dtype=np.float64) / 1e3
log = run.flow_log
pos = 0
for it in range(len(log)):
    ncross, nself = int(log[it, 1]), int(log[it, 2])
    nbar = 2 + 3 * ncross + 2 * nself + 2  # stats, pack, asym, sym, end, finalize
    st = t[pos:pos + 2 * nbar]
    if len(st) < 2 * nbar:
        break
    arr, rel = st[0::2], st[1::2]
    gap = (st[0] - t[pos - 1]) if pos else 0.0
    a0, a1 = 2, 2 + 3 * ncross
    s1 = a1 + 2 * nself
    print(f"flow {it:3d}: cross {ncross:2d} self {nself:2d} | kernel {rel[-1] - arr[0] + 0:7.1f} us"
          f" (from first barrier) | stats+pack {rel[1] - arr[0]:5.1f} | asym {rel[a1 - 1] - rel[1]:6.1f}"
          f" ({(rel[a1 - 1] - rel[1]) / max(ncross, 1):5.1f}/it) | sym {rel[s1 - 1] - rel[a1 - 1]:5.1f}"
          f" | end {rel[-1] - rel[s1 - 1]:5.1f} | gap before {gap:6.1f}")
    pos += 2 * nbar

# per-phase critical path of the asymmetric iterations (release-to-release)
pos = 0
acc = np.zeros(3)
cnt = 0
sym = np.zeros(2)
scnt = 0
for it in range(len(log)):
    ncross, nself = int(log[it, 1]), int(log[it, 2])
    nbar = 2 + 3 * ncross + 2 * nself + 2
    st = t[pos:pos + 2 * nbar]
    if len(st) < 2 * nbar:
        break
    rel = st[1::2]
    for k in range(ncross):
        b = 2 + 3 * k
        acc += [rel[b] - rel[b - 1], rel[b + 1] - rel[b], rel[b + 2] - rel[b + 1]]
        cnt += 1
    for k in range(nself):
        b = 2 + 3 * ncross + 2 * k
        sym += [rel[b] - rel[b - 1], rel[b + 1] - rel[b]]
        scnt += 1
    pos += 2 * nbar
print(f"asym per-iteration critical path (us): sweepA {acc[0]/cnt:.2f} sweepB(+mergeA) {acc[1]/cnt:.2f} "
      f"mergeB+err {acc[2]/cnt:.2f}  (n={cnt})")
print(f"sym per-iteration (us): sweep {sym[0]/scnt:.2f} merge {sym[1]/scnt:.2f} (n={scnt})")
