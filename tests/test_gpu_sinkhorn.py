"""Sinkhorn / entropic OT on the GPU vs the reference (golden) and the oracle.

Known-answer tests follow the reference's test_sinkhorn.py (cited per test);
parity tests use the golden vectors made by the reference itself and the
north_star tolerance: flows and potentials within 1e-4 relative (inf-norm),
fp32 vs the reference's float64.
"""

from __future__ import annotations

import itertools

import numpy as np
import pytest

import paper_2511_11514_b200 as fc
from fcb_testutil import load_golden, rel_inf
from oracle import flowcover_oracle as O
from paper_2511_11514_b200.sinkhorn import lse_sweep

pytestmark = pytest.mark.gpu
FLOW_TOL = 1e-4  # north_star: per-iteration flow fields / potentials


def random_pair(seed, n=8, m=7, dim=2):
    rng = np.random.default_rng(seed)
    return rng.random((n, dim)), rng.random((m, dim))


def _cfg(c, precision="auto"):
    return fc.SinkhornConfig(omega="auto" if c[0] == 0.0 else float(c[0]), max_iters=int(c[1]),
                             tol=float(c[2]), precision=precision)


# ---- golden parity ---------------------------------------------------------
@pytest.mark.parametrize("precision", ["auto", "float32", "float64"])
def test_entropic_ot_golden(precision):
    g = load_golden("ot_cases.npz")
    for k in range(int(g["ncases"])):
        X, Y, c = g[f"c{k}_X"], g[f"c{k}_Y"], g[f"c{k}_cfg"]
        cfg = _cfg(c, precision)
        if precision == "float32" and c[2] < 1e-7:
            continue  # fp32 cannot certify tol < 1e-7 (see _precision.py)
        sol = fc.entropic_ot(X, Y, cfg)
        scal = g[f"c{k}_scal"]
        tol = FLOW_TOL if (precision == "float32" or (precision == "auto" and X.shape[0] * Y.shape[0] >= 1 << 20)) else 1e-9
        assert sol.omega == pytest.approx(scal[4], rel=1e-12)
        if int(scal[1]) == int(cfg.max_iters) or sol.iters_used == int(scal[1]):
            assert rel_inf(sol.f, g[f"c{k}_f"]) <= tol, (k, rel_inf(sol.f, g[f"c{k}_f"]))
            assert rel_inf(sol.g, g[f"c{k}_g"]) <= tol, k
        assert abs(sol.iters_used - int(scal[1])) <= (0 if tol < 1e-6 else 1), k
        assert sol.converged == bool(scal[2]) or abs(sol.marginal_error - cfg.tol) < 0.05 * cfg.tol
        assert sol.cost == pytest.approx(scal[0], rel=max(tol, 1e-10), abs=1e-12)
        if f"c{k}_plan" in g:
            # exp((f+g-C)/w) amplifies potential errors by 1/w
            rtol = 1e-8 if tol < 1e-6 else 1e-3
            np.testing.assert_allclose(sol.plan(), g[f"c{k}_plan"], rtol=rtol, atol=1e-12)


@pytest.mark.parametrize("precision", ["float32", "float64"])
def test_single_sweep_golden(precision):
    g = load_golden("ot_cases.npz")
    L = lse_sweep(g["sweep_X"], g["sweep_Y"], g["sweep_pot"], float(g["sweep_omega"]), precision)
    assert rel_inf(L, g["sweep_L"]) <= (2e-6 if precision == "float32" else 1e-13)


def test_flow_golden_and_warm_state():
    g = load_golden("flow_cases.npz")
    for k in range(int(g["ncases"])):
        X, Y, c = g[f"c{k}_X"], g[f"c{k}_Y"], g[f"c{k}_cfg"]
        cfg = _cfg(c)
        warm = fc.SinkhornWarmState()
        first = fc.sinkhorn_flow(X, fc.SamplePoints(Y), cfg, warm=warm)
        assert rel_inf(first.a, g[f"c{k}_a"]) <= FLOW_TOL, (k, rel_inf(first.a, g[f"c{k}_a"]))
        second = fc.sinkhorn_flow(g[f"c{k}_X2"], fc.SamplePoints(Y), cfg, warm=warm)
        assert rel_inf(second.a, g[f"c{k}_a2"]) <= FLOW_TOL, k
        # the golden warm state is the one left by the second call
        assert rel_inf(warm.f, g[f"c{k}_warm_f"]) <= FLOW_TOL, (k, rel_inf(warm.f, g[f"c{k}_warm_f"]))
        assert rel_inf(warm.p, g[f"c{k}_warm_p"]) <= FLOW_TOL, k
        assert first.converged == bool(g[f"c{k}_scal"][0])
        if f"c{k}_div" in g:
            # a difference of three costs: fp32 cases keep ~1e-6 relative
            # (the north_star bar for coverage metrics is 1%)
            d = fc.sinkhorn_divergence(X, Y, cfg)
            assert d == pytest.approx(float(g[f"c{k}_div"]), rel=1e-4, abs=1e-9)


def test_fp32_flow_vs_oracle_at_config2_shape():
    """T=2000 states x M=1e4 targets (BASELINE configs[1] shape), fp32 kernels."""
    g = load_golden("flow_cases.npz")
    k = int(g["ncases"]) - 1
    X, Y = g[f"c{k}_X"], g[f"c{k}_Y"]
    assert X.shape == (2000, 2) and Y.shape == (10_000, 2)
    out = fc.sinkhorn_flow(X, fc.SamplePoints(Y), fc.SinkhornConfig(precision="float32"))
    assert rel_inf(out.a, g[f"c{k}_a"]) <= FLOW_TOL


def test_results_are_deterministic():
    X, Y = random_pair(3, 1500, 2500)
    a = fc.sinkhorn_flow(X, fc.SamplePoints(Y), fc.SinkhornConfig(precision="float32")).a
    b = fc.sinkhorn_flow(X, fc.SamplePoints(Y), fc.SinkhornConfig(precision="float32")).a
    assert np.array_equal(a, b)


# ---- reference known-answer tests (test_sinkhorn.py) -----------------------
def test_one_on_one_coupling_is_forced():  # test_sinkhorn.py:35-39
    sol = fc.entropic_ot(np.zeros((1, 2)), np.ones((1, 2)), fc.SinkhornConfig(omega=0.5))
    np.testing.assert_allclose(sol.plan(), [[1.0]], rtol=1e-15)
    assert sol.cost == pytest.approx(2.0, abs=1e-12)
    assert sol.converged


def test_identical_points_give_near_identity_plan():  # :42-50
    X = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0], [0.5, 0.5]])
    cfg = fc.SinkhornConfig(omega=1e-3, max_iters=50_000, tol=1e-10)
    sol = fc.entropic_ot(X, X, cfg)
    assert sol.converged
    P = sol.plan()
    np.testing.assert_allclose(P, np.eye(5) / 5, atol=1e-4)
    assert np.abs(P.sum(axis=1) - 0.2).max() <= cfg.tol * 1.01
    assert np.abs(P.sum(axis=0) - 0.2).max() <= cfg.tol * 1.01


def test_two_point_line_matches_identity_matching():  # :53-58
    X = np.array([[0.0], [1.0]])
    sol = fc.entropic_ot(X, X.copy(), fc.SinkhornConfig(omega=1e-3, max_iters=100_000, tol=1e-12))
    np.testing.assert_allclose(sol.plan(), [[0.5, 0.0], [0.0, 0.5]], atol=1e-3)
    assert abs(sol.cost) <= 1e-2


def test_unconverged_flag_is_honest():  # :61-66
    X, Y = random_pair(0)
    sol = fc.entropic_ot(X, Y, fc.SinkhornConfig(omega=0.01, max_iters=1, tol=1e-12))
    assert not sol.converged and sol.iters_used == 1 and sol.marginal_error > 1e-12


def test_rejects_non_finite_points():  # :69-72
    with pytest.raises(Exception, match="finite"):
        fc.entropic_ot(np.array([[0.0, np.nan]]), np.zeros((1, 2)))


def test_small_instances_match_assignment_lp():  # :75-85
    rng = np.random.default_rng(4)
    cfg = fc.SinkhornConfig(omega=1e-4, max_iters=5000, tol=1e-5)
    for n in (3, 4):
        X, Y = rng.random((n, 2)), rng.random((n, 2))
        C = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1)
        lp = min(C[range(n), perm].sum() / n for perm in itertools.permutations(range(n)))
        assert abs(fc.entropic_ot(X, Y, cfg).cost - lp) <= 0.01 * lp


def test_self_divergence_vanishes():  # :111-113
    X, _ = random_pair(1, n=20)
    assert abs(fc.sinkhorn_divergence(X, X, fc.SinkhornConfig(omega=0.05, tol=1e-10))) <= 1e-6


def test_divergence_axioms():  # :116-125
    rng = np.random.default_rng(123)
    cfg = fc.SinkhornConfig(omega=0.05, max_iters=20_000, tol=1e-11)
    for _ in range(8):
        X = rng.random((int(rng.integers(2, 13)), 2))
        Y = rng.random((int(rng.integers(2, 13)), 2))
        sxy = fc.sinkhorn_divergence(X, Y, cfg)
        assert sxy >= -1e-9
        assert abs(sxy - fc.sinkhorn_divergence(Y, X, cfg)) <= 1e-9


def test_rigid_shift_recovers_squared_distance():  # :128-133
    gr = np.linspace(0.0, 1.0, 16)
    X = np.array([(a, b) for a in gr for b in gr])
    S = fc.sinkhorn_divergence(X, X + np.array([0.5, 0.0]),
                               fc.SinkhornConfig(omega=0.01, max_iters=50_000, tol=1e-9))
    assert abs(S - 0.25) <= 0.025


def test_flow_vanishes_at_targets():  # :139-145
    X, _ = random_pair(2, n=25)
    out = fc.sinkhorn_flow(X, fc.SamplePoints(X.copy()), fc.SinkhornConfig(omega=0.05, tol=1e-9))
    assert np.abs(out.a).max() <= 1e-5 and out.converged


def test_single_pair_flow_points_at_target():  # :148-152
    x, y = np.array([[0.3, -0.2]]), np.array([[1.0, 0.6]])
    out = fc.sinkhorn_flow(x, fc.SamplePoints(y), fc.SinkhornConfig(omega=0.5))
    np.testing.assert_allclose(out.a, 2.0 * (y - x), atol=1e-9)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_flow_matches_finite_differences(seed):  # :155-171
    X, Y = random_pair(seed)
    cfg = fc.SinkhornConfig(omega=0.05, max_iters=50_000, tol=1e-10)
    a = fc.sinkhorn_flow(X, fc.SamplePoints(Y), cfg).a
    eps = 1e-5
    for i in range(X.shape[0]):
        for j in range(X.shape[1]):
            Xp, Xm = X.copy(), X.copy()
            Xp[i, j] += eps
            Xm[i, j] -= eps
            fd = (fc.sinkhorn_divergence(Xp, Y, cfg) - fc.sinkhorn_divergence(Xm, Y, cfg)) / (2 * eps)
            assert abs(-a[i, j] - fd) <= 1e-3 * max(abs(fd), 1e-8)


def test_flow_step_descends_divergence():  # :174-183
    rng = np.random.default_rng(9)
    cfg = fc.SinkhornConfig(omega=0.05, max_iters=50_000, tol=1e-10)
    for _ in range(5):
        X, Y = rng.random((20, 2)), rng.random((20, 2))
        a = fc.sinkhorn_flow(X, fc.SamplePoints(Y), cfg).a
        assert fc.sinkhorn_divergence(X + 1e-3 * a, Y, cfg) < fc.sinkhorn_divergence(X, Y, cfg)


def test_flow_error_on_gross_violation():  # :186-193
    rng = np.random.default_rng(3)
    X, Y = rng.random((12, 2)), rng.random((15, 2)) + 10.0
    with pytest.raises(fc.FlowError, match="marginal"):
        fc.sinkhorn_flow(X, fc.SamplePoints(Y), fc.SinkhornConfig(omega=0.01, max_iters=1, tol=1e-14))


def test_flow_flags_mild_violation_without_raising():  # :196-207
    rng = np.random.default_rng(3)
    X, Y = rng.random((12, 2)), rng.random((15, 2)) + 10.0
    probe = fc.entropic_ot(X, Y, fc.SinkhornConfig(omega=0.01, max_iters=1, tol=1e-14))
    tol = probe.marginal_error / 50
    out = fc.sinkhorn_flow(X, fc.SamplePoints(Y), fc.SinkhornConfig(omega=0.01, max_iters=1, tol=tol))
    assert not out.converged and out.marginal_error > tol


def test_warm_start_reproduces_cold_result():  # :210-219
    X, Y = random_pair(6, n=30, m=30)
    cfg = fc.SinkhornConfig(omega=0.05, max_iters=50_000, tol=1e-10)
    t = fc.SamplePoints(Y)
    cold = fc.sinkhorn_flow(X, t, cfg).a
    warm = fc.SinkhornWarmState()
    first = fc.sinkhorn_flow(X, t, cfg, warm=warm).a
    second = fc.sinkhorn_flow(X, t, cfg, warm=warm).a
    assert np.array_equal(first, cold)
    np.testing.assert_allclose(second, cold, atol=1e-8)


def test_auto_omega_matches_mean_squared_distance():  # :236-241
    X, Y = random_pair(5)
    sq = ((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1)
    assert np.isclose(fc.resolve_omega("auto", X, Y), 0.05 * sq.mean())
    assert fc.resolve_omega(0.3, X, Y) == 0.3


def test_ragged_and_tiny_shapes():
    """Sizes that are not multiples of any tile: 1, 7, 8, 9, 257, 1025 points."""
    for n, m in [(1, 1), (1, 9), (7, 1), (8, 8), (9, 257), (257, 1025), (1025, 3)]:
        X, Y = random_pair(n * 31 + m, n, m)
        cfg = fc.SinkhornConfig(omega=0.05, max_iters=200, tol=1e-9)
        a = fc.sinkhorn_flow(X, fc.SamplePoints(Y), cfg).a
        ref, _, _ = O.sinkhorn_flow(X, Y, 0.05, 200, 1e-9)
        assert rel_inf(a, ref) <= 1e-8, (n, m)
        f32 = fc.entropic_ot(X, Y, fc.SinkhornConfig(omega=0.05, max_iters=30, tol=1e-300,
                                                     precision="float32"))
        r = O.entropic_ot(X, Y, 0.05, 30, 1e-300)
        scale = max(np.abs(r["f"]).max(), np.abs(r["g"]).max())  # f may vanish (n = 1)
        assert np.abs(f32.f - r["f"]).max() <= FLOW_TOL * scale, (n, m)
        assert np.abs(f32.g - r["g"]).max() <= FLOW_TOL * scale, (n, m)


# ---- OT(Y, Y) cache of the divergence ---------------------
def _div_call(name, X, Y, omega, prec, cache=None):
    from paper_2511_11514_b200 import _dev, _lib
    lib = _lib.load()
    n, d = X.shape
    m = Y.shape[0]
    Xd, Yd = _dev.f64(X), _dev.f64(Y)
    out = _dev.empty((4,))
    ws = _dev.Workspace.get(lib.fcb_sinkhorn_divergence_workspace_bytes(prec, n, m, d), "t_div")
    args = [prec, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d, omega, 1000, 1e-6, _dev.ptr(out), None]
    if cache is not None:
        args.append(_dev.ptr(cache))
    _lib.call(name, *args, _dev.ptr(ws), ws.numel(), _dev.stream(), what=name)
    return out.cpu().numpy()


@pytest.mark.parametrize("prec", [0, 1])
def test_divergence_yy_cache_bit_identical(prec):
    """The cached call skips the M x M self solve when omega and m match, and
    returns exactly the uncached values; auto omega on a moved X misses."""
    import torch
    from paper_2511_11514_b200 import _lib
    rng = np.random.default_rng(5)
    Y = rng.random((900, 2))
    cache = torch.zeros(5, dtype=torch.float64, device="cuda")
    p = _lib.FCB_FP64 if prec else _lib.FCB_FP32
    for k, omega in enumerate([0.05, 0.05, 0.05]):
        X = rng.random((300 + 50 * k, 2))
        ref = _div_call("fcb_sinkhorn_divergence", X, Y, omega, p)
        got = _div_call("fcb_sinkhorn_divergence_cached", X, Y, omega, p, cache)
        assert np.array_equal(ref, got), (k, ref, got)
        c = cache.cpu().numpy()
        assert c[0] == 1.0 and c[1] > 0 and c[3] == 900 and c[4] == k  # hits so far
    # auto omega: resolved from X's moments, so a different X misses
    hits = float(cache[4])
    X = rng.random((300, 2)) * 0.5
    ref = _div_call("fcb_sinkhorn_divergence", X, Y, 0.0, p)
    got = _div_call("fcb_sinkhorn_divergence_cached", X, Y, 0.0, p, cache)
    assert np.array_equal(ref, got)
    assert float(cache[4]) == hits
    # a different m never hits
    Y2 = Y[:700]
    ref = _div_call("fcb_sinkhorn_divergence", X, Y2, 0.05, p)
    got = _div_call("fcb_sinkhorn_divergence_cached", X, Y2, 0.05, p, cache)
    assert np.array_equal(ref, got) and float(cache[4]) == hits and float(cache[3]) == 700


def test_plan_metric_with_fixed_omega_uses_cache():
    """plan() with a numeric omega and an in-loop metric: every metric value
    equals the public sinkhorn_divergence of that iteration's trajectory."""
    model = fc.single_integrator_2d()
    q = fc.benchmark_mixture(2)
    scfg = fc.SinkhornConfig(omega=0.02, precision="float64")
    cfg = fc.PlanConfig(method="sinkhorn", eta=60.0, max_iterations=4, convergence_tol=0.0,
                        metric_interval=2, metric_samples=400, seed=0, sinkhorn=scfg)
    tg = fc.SamplePoints(q.sample(600, [0, 2]))
    res = fc.plan(model, tg, fc.Discretization(0.05, 300, np.array([0.1, 0.1])), cfg)
    draws = tg.sample(400, [0, 3])
    final = fc.coverage_metric(res.trajectory.S, model, draws, scfg)
    assert res.metric_iterations[-1] == 4
    assert abs(res.metric_values[-1] - final) <= 1e-12 * max(1.0, abs(final))
