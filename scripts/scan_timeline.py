"""Per-block phase stamps of the one-launch affine scan (FCB_SCAN_TL builds).

    FCB_LIB_PATH=build_variants/scantl/libflowcover_b200.so python scripts/scan_timeline.py [T n m]

Marks: 0 start, 1 eta in-block scan done, 2 eta look-back done, 3 eta entry
known, 4 eta re-walk done, 5..8 the same for z, 9 end.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _lib  # noqa: E402

T, n, m = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (2000, 4, 2)
rng = np.random.default_rng(0)
A = 0.2 * rng.normal(size=(T, n, n)) - 0.5 * np.eye(n)
B = rng.normal(size=(T, n, m))
a = np.cumsum(rng.normal(scale=0.1, size=(T, n)), axis=0)
lib = _lib.load()
lib.fcb_debug_scan_timeline.argtypes = [ctypes.c_void_p]
lib.fcb_debug_scan_timeline.restype = ctypes.c_int
buf = (ctypes.c_ulonglong * (128 * 16))()
for rep in range(3):
    fc.solve_flow_lqr(fc.LtvSystem(A=A, B=B, dt=0.05), a, fc.LqrWeights(Q=np.eye(n), R=0.1 * np.eye(m)))
    torch.cuda.synchronize()
k = lib.fcb_debug_scan_timeline(buf)
t = np.array(buf[:k], dtype=np.float64).reshape(128, 16)
nb = (T + 127) // 128
t = t[:nb, :13]
t0 = t[:, 0].min()
print(f"T={T} n={n} m={m} blocks={nb}; microseconds since the first block started")
print("blk " + " ".join(f"{i:>7d}" for i in range(13)))
for b in range(nb):
    print(f"{b:3d} " + " ".join(f"{(v - t0) / 1e3:7.2f}" for v in t[b]))
