"""Device time of cold vs warm-started config-4 Sinkhorn flows (one GPU).

    python scripts/flow_cold_warm.py

X: the initial aircraft rollout (what a planner's first flow sees) and the
same X moved by a small step (what a later, warm flow sees)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _dev, _lib  # noqa: E402

m = fc.aircraft_3d()
T, M = 100_000, 1_000_000
U0 = fc.initial_controls(fc.PlanConfig(method="sinkhorn", seed=0), m, T)
S = fc.rollout(m, fc.default_start(m), U0, 0.05)
X = m.project_states(S[1:])
Y = fc.benchmark_mixture(3).sample(M, [0, 2])
lib = _lib.load()
Xd, Yd = _dev.f64(X), _dev.f64(Y)
n, d = X.shape
prec = _lib.FCB_FP32
ws = _dev.Workspace.get(lib.fcb_sinkhorn_flow_workspace_bytes(prec, n, M, d), "cw")
wf, wp = _dev.zeros((n,)), _dev.zeros((n,))
wv = torch.zeros(2, dtype=torch.int32, device="cuda")
flow, fstat = _dev.zeros((n, d)), _dev.zeros((8,))
print(f"X extent {np.ptp(X, axis=0)}, omega ~ {0.05 * ((X ** 2).sum(1).mean()):.3e}")


def run(Xdev, warm):
    if not warm:
        wv.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = lib.fcb_sinkhorn_flow(prec, _dev.ptr(Xdev), n, _dev.ptr(Yd), M, d, 0.0, 1000, 1e-6,
                               _dev.ptr(wf), _dev.ptr(wp), _dev.ptr(wv), _dev.ptr(flow),
                               _dev.ptr(fstat), None, 0, None, 0.0, _dev.ptr(ws), ws.numel(),
                               _dev.stream())
    _lib.check(rc, "flow")
    e1.record()
    e1.synchronize()
    st = fstat.cpu().numpy()
    pairs = 2 * st[5] * n * M + st[6] * n * n
    ms = e0.elapsed_time(e1)
    return ms, int(st[5]), int(st[6]), pairs / (ms * 1e-3)


for label, Xdev, warm in (("cold", Xd, False), ("cold", Xd, False), ("warm same X", Xd, True),
                          ("warm same X", Xd, True)):
    ms, ka, ks, rate = run(Xdev, warm)
    print(f"{label:12s} {ms:8.1f} ms  inner {ka}/{ks}  {rate:.3e} pair/s", flush=True)
