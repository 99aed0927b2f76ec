"""Phase timeline of one persistent asymmetric solve (FCB_TIMELINE builds).

    FCB_LIB_PATH=build_variants/tl/libflowcover_b200.so python scripts/timeline.py [n m iters]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11514_b200 import _dev, _lib  # noqa: E402
from paper_2511_11514_b200.sinkhorn import _resolve_on_device  # noqa: E402

n, m, iters = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (2000, 10000, 5)
rng = np.random.default_rng(0)
X, Y = rng.random((n, 2)), rng.random((m, 2))
Xd, Yd = _dev.f64(X), _dev.f64(Y)
scal = _resolve_on_device(0, 0, Xd, n, Yd, m, 2, 0.0)
f, g, rs = _dev.empty((n,)), _dev.empty((m,)), _dev.empty((n,))
stat, bary = _dev.empty((4,)), _dev.empty((n, 3))
lib = _lib.load()
ws = _dev.Workspace.get(lib.fcb_ot_workspace_bytes(0, 0, n, m, 2), "p")
buf = (ctypes.c_ulonglong * 8192)()
for rep in range(3):
    lib.fcb_debug_timeline(buf, 8192)
    _lib.call("fcb_ot_solve", 0, 0, _dev.ptr(Xd), n, _dev.ptr(Yd), m, 2, _dev.ptr(scal), iters,
              1e-300, None, _dev.ptr(f), _dev.ptr(g), _dev.ptr(rs), _dev.ptr(stat), _dev.ptr(bary),
              None, _dev.ptr(ws), ws.numel(), _dev.stream())
    torch.cuda.synchronize()
    k = lib.fcb_debug_timeline(buf, 8192)
t = np.array(buf[:k], dtype=np.float64)
t -= t[0]
print(f"{k} stamps; total {t[-1]/1e3:.1f} us for {iters} iterations")
if os.environ.get("FCB_TL_RAW"):
    for i in range(1, k):
        print(f"stamp {i:4d}: +{(t[i] - t[i - 1]) / 1e3:7.2f} us  (at {t[i] / 1e3:8.2f})")
    sys.exit(0)
names = ["pack", "sweepA", "mergeA", "sweepB", "mergeB"]
# stamps come in (arrive, release) pairs per barrier
prev_rel = 0.0
for b in range(k // 2):
    arr, rel = t[2 * b], t[2 * b + 1]
    phase = names[0] if b == 0 else names[1 + (b - 1) % 4]
    print(f"barrier {b:3d} after {phase:7s}: work {(arr - prev_rel)/1e3:7.2f} us   wait {(rel - arr)/1e3:6.2f} us")
    prev_rel = rel
