"""Phase timeline of median_cluster_kernel (build with -DMCL_TL), n=500 d=2."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _lib  # noqa: E402

X = np.random.default_rng(0).random((int(sys.argv[1]) if len(sys.argv) > 1 else 500, 2))
for _ in range(3):
    fc.median_bandwidth(X)
lib = _lib.load()
buf = (ctypes.c_ulonglong * 128)()
lib.fcb_debug_mcl_timeline.argtypes = [ctypes.c_void_p]
print("rc", lib.fcb_debug_mcl_timeline(ctypes.addressof(buf)))
for who in (0, 1):
    t = [buf[who * 64 + k] for k in range(64)]
    t0 = t[0]
    names = ["start"] + [f"p{p}.{n}" for p in range(6) for n in ("begin", "scanned", "syncA", "reduced", "syncB", "syncC")]
    line = []
    for k in list(range(37)) + [42, 40, 41]:
        if t[k]:
            line.append(f"{(names[k] if k < 37 else {40: "end0", 41: "end1", 42: "xloaded"}[k])}={(t[k] - t0) / 1e3:.2f}")
    print("CTA", "0" if who == 0 else "last", " ".join(line))
