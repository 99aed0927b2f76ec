"""Out-of-bounds write guards for the C ABI (stand-in for compute-sanitizer).

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a
reset), so every output buffer and workspace handed to the entry points here
sits between two guard bands filled with a sentinel; after each call the bands
must be untouched.  Shapes are ragged on purpose (not multiples of the tile,
quad, chunk or warp sizes) and cover each kernel family on the paths the
BASELINE configs take.  Results themselves are checked by the parity tests.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest
import torch

import paper_2511_11514_b200 as fc
from paper_2511_11514_b200 import _dev, _lib
from paper_2511_11514_b200.dynamics import device_model

pytestmark = pytest.mark.gpu
PAD = 4096  # bytes of guard on each side
SENT = 0xA5


class Guarded:
    """A device buffer with guard bands (uint8 storage, typed view in the middle)."""

    def __init__(self, shape, dtype=torch.float64, init=None):
        esz = torch.tensor([], dtype=dtype).element_size()
        n = int(np.prod(shape)) if len(shape) else 1
        self.raw = torch.full((2 * PAD + n * esz,), SENT, dtype=torch.uint8, device="cuda")
        self.view = self.raw[PAD:PAD + n * esz].view(dtype).view(shape)
        if init is not None:
            self.view.copy_(torch.as_tensor(init, dtype=dtype))

    @property
    def ptr(self):
        return ctypes.c_void_p(self.view.data_ptr())

    def intact(self) -> bool:
        torch.cuda.synchronize()
        lo, hi = self.raw[:PAD], self.raw[-PAD:]
        return bool((lo == SENT).all() and (hi == SENT).all())


def ws(nbytes):
    return Guarded((max(int(nbytes), 1),), torch.uint8)


def check(*bufs):
    bad = [i for i, b in enumerate(bufs) if not b.intact()]
    assert not bad, f"guard band overwritten for buffer(s) {bad}"


def lib():
    return _lib.load()


@pytest.mark.parametrize("n,m,d,prec,resident", [
    (701, 1533, 2, 0, "1"), (701, 1533, 2, 0, "0"), (301, 907, 3, 0, "1"),
    (301, 907, 3, 0, "0"), (77, 130, 1, 1, "0"), (5003, 40_009, 2, 0, "0"),
])
def test_sinkhorn_flow_guards(monkeypatch, n, m, d, prec, resident):
    monkeypatch.setenv("FCB_RESIDENT", resident)
    q = fc.benchmark_mixture(2 if d != 3 else 3) if d > 1 else None
    rng = np.random.default_rng(n)
    X = rng.random((n, d)) if q is None else q.sample(n, [1, 2])
    Y = rng.random((m, d)) if q is None else q.sample(m, [0, 2])
    Xd, Yd = _dev.f64(X), _dev.f64(Y)
    L = lib()
    flow, fstat = Guarded((n, d)), Guarded((8,))
    wf, wp, wv = Guarded((n,)), Guarded((n,)), Guarded((2,), torch.int32, [0, 0])
    w = ws(L.fcb_sinkhorn_flow_workspace_bytes(prec, n, m, d))
    for _ in range(2):  # cold, then warm
        rc = L.fcb_sinkhorn_flow(prec, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d, 0.0, 1000, 1e-6, wf.ptr,
                                 wp.ptr, wv.ptr, flow.ptr, fstat.ptr, None, 0, None, 0.0, w.ptr,
                                 w.view.numel(), _dev.stream())
        _lib.check(rc, "fcb_sinkhorn_flow")
        check(flow, fstat, wf, wp, wv, w)


@pytest.mark.parametrize("mode", [0, 1])
def test_ot_solve_and_sweep_guards(mode):
    rng = np.random.default_rng(3)
    n, m, d = 1029, 2051, 3
    Xd, Yd = _dev.f64(rng.random((n, d))), _dev.f64(rng.random((m, d)))
    L = lib()
    scal = Guarded((16,))
    wo = ws(L.fcb_omega_workspace_bytes(n, m))
    _lib.check(L.fcb_resolve_omega(mode, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d, 0.0, scal.ptr,
                                   wo.ptr, wo.view.numel(), _dev.stream()), "omega")
    f, g, rs, stat, bary = (Guarded((n,)), Guarded((m,)), Guarded((n,)), Guarded((4,)),
                            Guarded((n, d + 1)))
    w = ws(L.fcb_ot_workspace_bytes(mode, 0, n, m, d))
    _lib.check(L.fcb_ot_solve(mode, 0, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d, scal.ptr, 50, 1e-6,
                              None, f.ptr, g.ptr if mode == 0 else None, rs.ptr, stat.ptr,
                              bary.ptr, None, w.ptr, w.view.numel(), _dev.stream()), "ot")
    check(scal, wo, f, g, rs, stat, bary, w)
    # one sharded-style sweep with the epilogue and a row estimate
    out, bl = Guarded((n,)), Guarded((n, d + 1))
    pot = _dev.f64(rng.normal(scale=0.01, size=m))
    est = _dev.f64(np.zeros(n))
    w2 = ws(L.fcb_lse_sweep_workspace_bytes(0, n, m, d))
    _lib.check(L.fcb_lse_sweep(0, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d, scal.ptr, _dev.ptr(pot),
                               _dev.ptr(est), -math.log(m), 1.0, -math.log(m), out.ptr, bl.ptr,
                               None, w2.ptr, w2.view.numel(), _dev.stream()), "lse_sweep")
    check(out, bl, w2)


@pytest.mark.parametrize("n,d,bw", [(613, 2, 0.0), (1501, 3, 0.01), (5, 2, 0.0)])
def test_stein_guards(n, d, bw):
    q = fc.benchmark_mixture(d) if d > 1 else None
    X = np.random.default_rng(n).random((n, d))
    if q is None:
        pytest.skip("mixtures are 2-D / 3-D")
    L = lib()
    Xd = _dev.f64(X)
    flow, fstat = Guarded((n, d)), Guarded((8,))
    w = ws(L.fcb_stein_flow_full_workspace_bytes(0, n, d))
    _lib.check(L.fcb_stein_flow_full(0, _dev.ptr(Xd), n, d, q.num_components,
                                     _dev.ptr(q.device_params()), bw, math.log(n + 1.0), flow.ptr,
                                     fstat.ptr, None, 0, None, 0.0, w.ptr, w.view.numel(),
                                     _dev.stream()), "stein")
    check(flow, fstat, w)


@pytest.mark.parametrize("name,T", [("single_integrator_2d", 1237), ("diff_drive", 1237),
                                    ("aircraft_3d", 20_011), ("double_integrator_2d", 129)])
def test_rollout_lqr_update_guards(name, T):
    model = fc.double_integrator_2d() if name == "double_integrator_2d" else fc.get_model(name)
    spec = device_model(model)
    ns, mc, d = model.state_dim, model.control_dim, model.workspace_dim
    L = lib()
    prm = spec.device_params(_dev.require_cuda())
    U = _dev.f64(1e-2 * np.random.default_rng(T).standard_normal((T, mc)))
    s0 = _dev.f64(fc.default_start(model) if name != "double_integrator_2d"
                  else np.array([0.1, 0.1, 0, 0]))
    P = _dev.f64(model.project_matrix)
    for method in (0, 1):
        S, X, status = Guarded((T + 1, ns)), Guarded((T, d)), Guarded((1,), torch.int32)
        w = ws(L.fcb_rollout_workspace_bytes(ns, T))
        _lib.check(L.fcb_rollout(spec.model_id, ns, mc, _dev.ptr(prm), _dev.ptr(s0), _dev.ptr(U),
                                 T, 0.05, S.ptr, d, _dev.ptr(P), X.ptr, status.ptr, None, 0,
                                 method, w.ptr, _dev.stream()), "rollout")
        check(S, X, status, w)
    wts = fc.workspace_weights(model.project_matrix, mc)
    Q, R = _dev.f64(wts.Q), _dev.f64(wts.R)
    flow = _dev.f64(1e-3 * np.random.default_rng(1).standard_normal((T, d)))
    Un, costs = Guarded((T, mc)), Guarded((3,))
    state = Guarded((8,), torch.int32, np.zeros(8))
    w = ws(L.fcb_plan_update_workspace_bytes(ns, mc, T))
    for mode in (0, 1):
        _lib.check(L.fcb_plan_update(spec.model_id, ns, mc, _dev.ptr(prm), S.ptr, _dev.ptr(U), T,
                                     0.05, d, _dev.ptr(P), _dev.ptr(flow), _dev.ptr(Q), _dev.ptr(R),
                                     1.0, None, Un.ptr, costs.ptr, state.ptr, mode, mode, w.ptr,
                                     w.view.numel(), _dev.stream()), "plan_update")
        check(Un, costs, state, w)
    # explicit-array LQR
    ltv = fc.linearize_along(model, _dev.host(S.view), _dev.host(U), 0.05)
    A, B = _dev.f64(ltv.A), _dev.f64(ltv.B)
    a = _dev.f64(1e-3 * np.random.default_rng(2).standard_normal((T, ns)))
    v, z, K, dff = Guarded((T, mc)), Guarded((T + 1, ns)), Guarded((T, mc, ns)), Guarded((T, mc))
    scal, st = Guarded((2,)), Guarded((1,), torch.int32)
    w = ws(L.fcb_lqr_workspace_bytes(ns, mc, T))
    _lib.check(L.fcb_lqr_solve(ns, mc, T, 0.05, _dev.ptr(A), _dev.ptr(B), _dev.ptr(Q), _dev.ptr(R),
                               _dev.ptr(a), v.ptr, z.ptr, K.ptr, dff.ptr, scal.ptr, st.ptr,
                               w.ptr, _dev.stream()), "lqr")
    check(v, z, K, dff, scal, st, w)


def test_gather_and_tour_guards():
    L = lib()
    rng = np.random.default_rng(5)
    src = _dev.f64(rng.random((1001, 3)))
    idx = torch.from_numpy(rng.integers(0, 1001, size=777).astype(np.int32)).cuda()
    out, status = Guarded((777, 3)), Guarded((1,), torch.int32)
    _lib.check(L.fcb_gather_rows(_dev.ptr(src), 1001, 3, _dev.ptr(idx), 777, out.ptr, status.ptr,
                                 _dev.stream()), "gather")
    check(out, status)
    assert int(status.view[0]) == -1
    pts = _dev.f64(rng.random((3, 333, 2)))
    starts = torch.tensor([0, 5, 332], dtype=torch.int32, device="cuda")
    order, moves = Guarded((3, 333), torch.int32), Guarded((3,), torch.int32)
    _lib.check(L.fcb_tsp_tours(_dev.ptr(pts), 3, 333, 2, _dev.ptr(starts), 3330, order.ptr,
                               moves.ptr, _dev.stream()), "tsp")
    check(order, moves)
    for b in range(3):
        assert sorted(order.view[b].tolist()) == list(range(333))


def test_sharded_step_guards():
    from paper_2511_11514_b200 import distributed as D

    rng = np.random.default_rng(6)
    n, m, d, R = 517, 1301, 3, 3
    X, Y = _dev.f64(rng.random((n, d))), _dev.f64(rng.random((m, d)))
    L = lib()
    ysum = Guarded((d + 2,))
    _lib.check(L.fcb_point_sums(_dev.ptr(Y), m, d, ysum.ptr, _dev.stream()), "sums")
    scal_x, scal_s, f, p = Guarded((16,)), Guarded((16,)), Guarded((n,)), Guarded((n,))
    ctl, eslot = Guarded((8,), torch.int32), Guarded((2,), torch.int64)
    _lib.check(L.fcb_shard_init(0, _dev.ptr(X), n, d, ysum.ptr, 0.0, None, None, None, scal_x.ptr,
                                scal_s.ptr, f.ptr, p.ptr, ctl.ptr, eslot.ptr, None,
                                _dev.stream()), "init")
    gath = _dev.f64(np.concatenate([np.c_[rng.normal(size=(n, 1)) - 3, rng.random((n, d))]
                                    for _ in range(R)]))
    fnext, rs, mass, ybar, stat = (Guarded((n,)), Guarded((n,)), Guarded((n,)), Guarded((n, d)),
                                   Guarded((4,)))
    _lib.check(L.fcb_shard_cross_merge(n, d, R, _dev.ptr(gath), scal_x.ptr, 1e-6, 3, f.ptr,
                                       fnext.ptr, rs.ptr, mass.ptr, ybar.ptr, ctl.ptr, eslot.ptr,
                                       stat.ptr, _dev.stream()), "merge")
    check(ysum, scal_x, scal_s, f, p, ctl, eslot, fnext, rs, mass, ybar, stat)
    chunk = (n + R - 1) // R
    lo, hi = D.shard_bounds(n, 1, R)
    Lb = _dev.f64(np.c_[rng.normal(size=(hi - lo, 1)), rng.random((hi - lo, d))])
    send = Guarded((chunk, d + 4))
    _lib.check(L.fcb_shard_self_rows(n, d, lo, hi - lo, _dev.ptr(Lb), scal_s.ptr, p.ptr, send.ptr,
                                     ctl.ptr, _dev.stream()), "self rows")
    check(send, p)
    parts = _dev.f64(rng.random((R, n, d + 1)))
    hstat = _dev.f64([0.02, np.nan, 0.0, 0.0])
    flow, fstat = Guarded((n, d)), Guarded((8,))
    w = ws(L.fcb_stein_combine_workspace_bytes(n))
    _lib.check(L.fcb_stein_combine(_dev.ptr(X), n, d, R, _dev.ptr(parts), _dev.ptr(hstat),
                                   flow.ptr, fstat.ptr, None, 0, None, 0.0, w.ptr, w.view.numel(),
                                   _dev.stream()), "combine")
    check(flow, fstat, w)


def test_cached_divergence_guards():
    rng = np.random.default_rng(8)
    n, m, d = 413, 977, 2
    Xd, Yd = _dev.f64(rng.random((n, d))), _dev.f64(rng.random((m, d)))
    L = lib()
    out, cache = Guarded((4,)), Guarded((5,), init=np.zeros(5))
    w = ws(L.fcb_sinkhorn_divergence_workspace_bytes(0, n, m, d))
    for _ in range(2):  # miss, then hit
        _lib.check(L.fcb_sinkhorn_divergence_cached(0, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d, 0.05,
                                                    200, 1e-6, out.ptr, None, cache.ptr, w.ptr,
                                                    w.view.numel(), _dev.stream()), "div_cached")
        check(out, cache, w)
    assert float(cache.view[4]) == 1.0


@pytest.mark.parametrize("T,bw", [(517, 0.0), (131, 0.03)])
def test_fused_stein_planner_guards(T, bw):
    """fcb_plan_fused_stein (sv_plan_kernel) with every output guarded, on
    the stored Riccati phase of a mode-0 update (as plan() runs it)."""
    model = fc.double_integrator_2d()
    spec = device_model(model)
    ns, mc, d = model.state_dim, model.control_dim, model.workspace_dim
    L = lib()
    dev = _dev.require_cuda()
    prm = spec.device_params(dev)
    q = fc.benchmark_mixture(2)
    s0 = _dev.f64(np.array([0.1, 0.1, 0.0, 0.0]))
    P = _dev.f64(model.project_matrix)
    wts = fc.workspace_weights(model.project_matrix, mc)
    Q, R = _dev.f64(wts.Q), _dev.f64(wts.R)
    maxit = 4
    U0 = Guarded((T, mc), init=1e-2 * np.random.default_rng(T).standard_normal((T, mc)))
    U1, S0, S1 = Guarded((T, mc)), Guarded((T + 1, ns)), Guarded((T + 1, ns))
    X, flow = Guarded((T, d)), Guarded((T, d))
    fstat, state = Guarded((8,)), Guarded((8,), torch.int32, np.zeros(8))
    flow_log, costs = Guarded((maxit, 4)), Guarded((maxit,))
    phase = Guarded((3,), torch.int64, np.zeros(3))
    upd = ws(L.fcb_plan_update_workspace_bytes(ns, mc, T))
    scratch = torch.zeros(8, dtype=torch.int32, device="cuda")
    z = lambda *s: _dev.zeros(s)  # noqa: E731
    _lib.check(L.fcb_plan_update(spec.model_id, ns, mc, _dev.ptr(prm), _dev.ptr(z(T + 1, ns)),
                                 _dev.ptr(z(T, mc)), T, 0.05, d, _dev.ptr(P), _dev.ptr(z(T, d)),
                                 _dev.ptr(Q), _dev.ptr(R), 0.1, None, _dev.ptr(z(T, mc)),
                                 _dev.ptr(z(maxit)), _dev.ptr(scratch), 0, 0, upd.ptr,
                                 upd.view.numel(), _dev.stream()), "plan_update")
    w = ws(L.fcb_plan_fused_stein_workspace_bytes(T, d, mc))
    rc = L.fcb_plan_fused_stein(spec.model_id, ns, mc, _dev.ptr(prm), _dev.ptr(s0), U0.ptr, U1.ptr,
                                S0.ptr, S1.ptr, T, 0.05, d, _dev.ptr(P), X.ptr, flow.ptr,
                                _dev.ptr(Q), _dev.ptr(R), 0.1, None, q.num_components,
                                _dev.ptr(q.device_params()), bw, math.log(T + 1.0), 0.0,
                                fstat.ptr, state.ptr, flow_log.ptr, costs.ptr, phase.ptr, 1, maxit,
                                upd.ptr, w.ptr, w.view.numel(), _dev.stream())
    _lib.check(rc, "plan_fused_stein")
    check(U0, U1, S0, S1, X, flow, fstat, state, flow_log, costs, phase, upd, w)
    st = state.view.cpu().numpy()
    assert st[0] == 0 and st[4] == maxit and st[5] == maxit  # flows, updates
