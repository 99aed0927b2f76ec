"""Per-iteration device time of the fp32 asymmetric / symmetric solve.

    python scripts/solve_bench.py            # config-sized shapes
    FCB_OT_CTAS_PER_SM=1 python scripts/solve_bench.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11514_b200 import _dev, _lib  # noqa: E402
from paper_2511_11514_b200.sinkhorn import _resolve_on_device  # noqa: E402

lib = _lib.load()


def bench(mode, n, m, iters, reps=3):
    rng = np.random.default_rng(0)
    X, Y = rng.random((n, 2)), rng.random((max(m, 1), 2))
    Xd, Yd = _dev.f64(X), _dev.f64(Y)
    mm = m if mode == _lib.FCB_OT_ASYM else 0
    scal = _resolve_on_device(mode, _lib.FCB_FP32, Xd, n, Yd, mm, 2, 0.0)
    f, g, rs = _dev.empty((n,)), _dev.empty((max(m, 1),)), _dev.empty((n,))
    stat, bary = _dev.empty((4,)), _dev.empty((n, 3))
    ws = _dev.Workspace.get(lib.fcb_ot_workspace_bytes(mode, _lib.FCB_FP32, n, mm, 2), "sb")
    best = 1e30
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("fcb_ot_solve", mode, _lib.FCB_FP32, _dev.ptr(Xd), n, _dev.ptr(Yd), mm, 2,
                  _dev.ptr(scal), iters, 1e-300, None, _dev.ptr(f), _dev.ptr(g), _dev.ptr(rs),
                  _dev.ptr(stat), None, None, _dev.ptr(ws), ws.numel(), _dev.stream())
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    pairs = (2 * n * m if mode == _lib.FCB_OT_ASYM else n * n) * iters
    print(f"{'asym' if mode == _lib.FCB_OT_ASYM else 'sym '} {n:>7d} x {m:>8d}: {best / iters:9.1f} us/iter"
          f"  {pairs / best * 1e-6:8.3f} Tpair/s")


for n, m, it in [(2000, 10000, 20), (10000, 100000, 10), (100000, 1000000, 2)]:
    bench(_lib.FCB_OT_ASYM, n, m, it)
for n, it in [(2000, 20), (10000, 10)]:
    bench(_lib.FCB_OT_SYM, n, 0, it)
