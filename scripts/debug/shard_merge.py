"""Debug: one fcb_shard_cross_merge call with R=3 synthetic shard partials."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
from paper_2511_11514_b200 import distributed as D  # noqa: E402
from shard_cpu_ops import CpuOps  # noqa: E402

for d in (1, 2):
    rng = np.random.default_rng(d)
    n, R = 1001, 3
    g = np.empty((R, n, d + 1))
    g[:, :, 0] = rng.normal(scale=3.0, size=(R, n)) - 5.0
    g[:, :, 1:] = rng.random((R, n, d))
    f0 = rng.normal(scale=0.01, size=n)
    for name, ops in (("gpu", D.DeviceOps()), ("cpu", CpuOps())):
        t = ops.tensor
        scal = t(np.r_[0.03, np.zeros(15)])
        f, fnext = t(f0), ops.zeros((n,))
        rs, mass, ybar = ops.zeros((n,)), ops.zeros((n,)), ops.zeros((n, d))
        ctl = ops.zeros((8,), dtype=torch.int32)
        eslot = ops.zeros((2,), dtype=torch.int64)
        stat = ops.zeros((4,))
        ops.cross_merge(n, d, R, t(g), scal, 1e-6, 5, f, fnext, rs, mass, ybar, ctl, eslot, stat)
        if name == "gpu":
            torch.cuda.synchronize()
        print(d, name, "ctl", ctl.cpu().tolist(), "stat", stat.cpu().tolist(), "eslot",
              eslot.cpu().tolist(), "f[:3]", f.cpu().numpy()[:3], "fnext[:3]", fnext.cpu().numpy()[:3],
              "f0[:3]", f0[:3])
