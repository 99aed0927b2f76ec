"""Profiling driver: the dominant kernels at BASELINE configs[1] shapes.

  python scripts/profile_ot.py phases     # per-phase device time of plan()
  python scripts/profile_ot.py solve      # asym solve replay (ncu target)
  python scripts/profile_ot.py sweep N M  # one fp32 LSE sweep of N x M pairs
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _dev, _lib  # noqa: E402
from paper_2511_11514_b200.sinkhorn import _resolve_on_device  # noqa: E402

S0 = np.array([0.1, 0.1, 0.0, 0.0])


def phases(iters=20):
    q = fc.benchmark_mixture(2)
    Y = q.sample(10_000, [0, 2])
    cfg = fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=iters, convergence_tol=0.0,
                        metric_interval=0)
    for _ in range(2):
        run = fc.plan_detailed(fc.double_integrator_2d(), fc.SamplePoints(Y),
                               fc.Discretization(0.05, 2000, S0), cfg)
    pt = run.result.phase_times
    print(f"iters={iters} total={pt.total*1e3:.1f}ms flow={pt.flow*1e3:.1f}ms "
          f"lqr={pt.lqr*1e3:.1f}ms rollout={pt.rollout*1e3:.1f}ms pairs={run.pairs:.3e}")
    lg = run.flow_log
    if lg is not None and len(lg):
        print(f"sinkhorn iterations per flow: cross mean {lg[:, 1].mean():.1f} max {lg[:, 1].max():.0f}"
              f" | self mean {lg[:, 2].mean():.1f} max {lg[:, 2].max():.0f}")


def solve(reps=5, n=2000, m=10_000, iters=10):
    rng = np.random.default_rng(0)
    X, Y = rng.random((n, 2)), rng.random((m, 2))
    Xd, Yd = _dev.f64(X), _dev.f64(Y)
    scal = _resolve_on_device(_lib.FCB_OT_ASYM, _lib.FCB_FP32, Xd, n, Yd, m, 2, 0.0)
    f, g, rs = _dev.empty((n,)), _dev.empty((m,)), _dev.empty((n,))
    stat, bary = _dev.empty((4,)), _dev.empty((n, 3))
    lib = _lib.load()
    ws = _dev.Workspace.get(lib.fcb_ot_workspace_bytes(0, 0, n, m, 2), "p")
    for _ in range(reps):
        _lib.call("fcb_ot_solve", 0, 0, _dev.ptr(Xd), n, _dev.ptr(Yd), m, 2, _dev.ptr(scal),
                  iters, 1e-300, None, _dev.ptr(f), _dev.ptr(g), _dev.ptr(rs), _dev.ptr(stat),
                  _dev.ptr(bary), None, _dev.ptr(ws), ws.numel(), _dev.stream())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("fcb_ot_solve", 0, 0, _dev.ptr(Xd), n, _dev.ptr(Yd), m, 2, _dev.ptr(scal),
              iters, 1e-300, None, _dev.ptr(f), _dev.ptr(g), _dev.ptr(rs), _dev.ptr(stat),
              _dev.ptr(bary), None, _dev.ptr(ws), ws.numel(), _dev.stream())
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    pairs = 2.0 * iters * n * m
    print(f"solve n={n} m={m} iters={iters}: {t*1e3:.3f} ms, {pairs/t/1e9:.1f} Gpair/s")


def sweep(n, m, reps=10):
    rng = np.random.default_rng(0)
    X, Y = rng.random((n, 2)), rng.random((m, 2))
    pot = rng.normal(scale=0.01, size=m)
    from paper_2511_11514_b200.sinkhorn import lse_sweep
    for _ in range(2):
        lse_sweep(X, Y, pot, 0.02, "float32")
    Xd, Yd, pd = _dev.f64(X), _dev.f64(Y), _dev.f64(pot)
    scal = _resolve_on_device(_lib.FCB_OT_SWEEP, _lib.FCB_FP32, Xd, n, Yd, m, 2, 0.02)
    out = _dev.empty((n,))
    lib = _lib.load()
    ws = _dev.Workspace.get(lib.fcb_ot_workspace_bytes(2, 0, n, m, 2), "p")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _lib.call("fcb_ot_solve", 2, 0, _dev.ptr(Xd), n, _dev.ptr(Yd), m, 2, _dev.ptr(scal), 1,
                  0.0, _dev.ptr(pd), _dev.ptr(out), None, None, None, None, None, _dev.ptr(ws),
                  ws.numel(), _dev.stream())
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / reps
    print(f"sweep {n}x{m}: {t*1e3:.3f} ms/launch, {n*m/t/1e9:.1f} Gpair/s")


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "phases":
        phases()
    elif what == "solve":
        solve()
    elif what == "sweep":
        sweep(int(sys.argv[2]), int(sys.argv[3]))


def lqr(T=2000, reps=5):
    rng = np.random.default_rng(0)
    n, m = 4, 2
    A = np.zeros((T, n, n)); A[:, 0, 2] = A[:, 1, 3] = 1.0
    B = np.zeros((T, n, m)); B[:, 2, 0] = B[:, 3, 1] = 1.0
    P = np.zeros((2, 4)); P[0, 0] = P[1, 1] = 1.0
    a = rng.normal(size=(T, 2)) @ P
    sys_ = fc.LtvSystem(A=A, B=B, dt=0.05)
    w = fc.workspace_weights(P, 2)
    for _ in range(reps):
        fc.solve_flow_lqr(sys_, a, w)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fc.solve_flow_lqr(sys_, a, w)
    print(f"lqr T={T}: {(time.perf_counter()-t0)/reps*1e3:.3f} ms per solve (incl. host copies)")


if __name__ == "__main__" and sys.argv[1] == "lqr":
    lqr(int(sys.argv[2]) if len(sys.argv) > 2 else 2000)
