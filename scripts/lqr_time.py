"""Time one planner LQR update (fcb_plan_update, mode 0: Riccati + affine phase)
for a nonlinear model at a long horizon, on one GPU.

    python scripts/lqr_time.py [model] [T] [reps]

Prints ms per update (CUDA events); run under ncu for the per-kernel split.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _dev, _lib  # noqa: E402
from paper_2511_11514_b200.dynamics import device_model  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "aircraft_3d"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
model = fc.get_model(name)
spec = device_model(model)
n_s, m_c, d = model.state_dim, model.control_dim, model.workspace_dim
rng = np.random.default_rng(0)
U = 1e-2 * rng.standard_normal((T, m_c))
S = fc.rollout(model, fc.default_start(model), U, 0.05)
flow = 1e-3 * rng.standard_normal((T, d))
w = fc.workspace_weights(model.project_matrix, m_c, 1.0, 0.1)
lib = _lib.load()
dev = _dev.require_cuda()
Sd, Ud, fd = _dev.f64(S), _dev.f64(U), _dev.f64(flow)
P, Q, R = _dev.f64(model.project_matrix), _dev.f64(w.Q), _dev.f64(w.R)
prm = spec.device_params(dev)
Un = _dev.zeros((T, m_c))
costs = _dev.zeros((reps + 4,))
state = torch.zeros(8, dtype=torch.int32, device=dev)
ws = _dev.Workspace.get(lib.fcb_plan_update_workspace_bytes(n_s, m_c, T), "upd")


def once(i):
    rc = lib.fcb_plan_update(spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(Sd), _dev.ptr(Ud), T,
                             0.05, d, _dev.ptr(P), _dev.ptr(fd), _dev.ptr(Q), _dev.ptr(R), 1.0, None,
                             _dev.ptr(Un), _dev.ptr(costs), _dev.ptr(state), i, 0, _dev.ptr(ws),
                             ws.numel(), _dev.stream())
    _lib.check(rc, "fcb_plan_update")


for i in range(2):
    once(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(reps):
    once(2 + i)
e1.record()
e1.synchronize()
print(f"{name} T={T}: {e0.elapsed_time(e1) / reps:.3f} ms per LQR update (mode 0); "
      f"state={state.tolist()} cost={float(costs[2]):.6e}")
