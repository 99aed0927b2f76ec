"""The planner's parallel rollouts (affine scan for linear models, two prefix
scans for the triangular nonlinear models) vs the sequential RK4 kernel."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2511_11514_b200 as fc
from fcb_testutil import rel_inf
from paper_2511_11514_b200 import _dev, _lib
from paper_2511_11514_b200.dynamics import device_model

pytestmark = pytest.mark.gpu


def _roll(model, s0, U, dt, method):
    spec = device_model(model)
    dev = _dev.require_cuda()
    T = U.shape[0]
    lib = _lib.load()
    ws = _dev.Workspace.get(lib.fcb_rollout_workspace_bytes(spec.state_dim, T), "test_roll")
    prm = spec.device_params(dev)
    s0d, Ud = _dev.f64(s0, dev), _dev.f64(U, dev)
    P = _dev.f64(model.project_matrix, dev)
    S = _dev.zeros((T + 1, spec.state_dim), device=dev)
    X = _dev.zeros((T, model.workspace_dim), device=dev)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.call("fcb_rollout", spec.model_id, spec.state_dim, spec.control_dim, _dev.ptr(prm),
              _dev.ptr(s0d), _dev.ptr(Ud), T, float(dt), _dev.ptr(S), model.workspace_dim,
              _dev.ptr(P), _dev.ptr(X), _dev.ptr(status), None, 0, method, _dev.ptr(ws),
              _dev.stream())
    return _dev.host(S), _dev.host(X), int(status.item())


@pytest.mark.parametrize("name", ["single_integrator_2d", "diff_drive", "aircraft_3d",
                                  "double_integrator_2d"])
@pytest.mark.parametrize("T", [1, 127, 128, 129, 3000, 20000])
def test_scan_rollout_matches_sequential(name, T):
    model = fc.double_integrator_2d() if name == "double_integrator_2d" else fc.get_model(name)
    rng = np.random.default_rng(T)
    U = rng.normal(scale=0.5, size=(T, model.control_dim))
    s0 = fc.default_start(model) if name != "double_integrator_2d" else np.array([0.1, 0.1, 0, 0])
    S0, X0, st0 = _roll(model, s0, U, 0.05, 0)
    S1, X1, st1 = _roll(model, s0, U, 0.05, 1)
    assert st0 == st1 == -1
    assert rel_inf(S1, S0) <= 1e-11
    assert rel_inf(X1, model.project_states(S0[1:])) <= 1e-11


@pytest.mark.parametrize("name", ["single_integrator_2d", "diff_drive"])
def test_scan_rollout_reports_first_nonfinite_step(name):
    model = fc.get_model(name)
    U = np.zeros((300, 2))
    U[137, 0] = 1e308
    U[138:, 0] = 1e308
    _, _, st0 = _roll(model, fc.default_start(model), U, 0.1, 0)
    _, _, st1 = _roll(model, fc.default_start(model), U, 0.1, 1)
    assert st0 == st1 and st0 > 0
