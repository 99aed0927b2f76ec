"""The on-device planner loop vs the reference's plan() (golden runs).

North_star tolerances: per-iteration flow fields within 1e-4 relative on
identical inputs; final trajectories and coverage metrics within 1%.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2511_11514_b200 as fc
from fcb_testutil import load_golden, rel_inf
from paper_2511_11514_b200.seeding import STREAM_METRIC, STREAM_REFERENCE

pytestmark = pytest.mark.gpu
DI_S0 = np.array([0.1, 0.1, 0.0, 0.0])


def test_config1_stein_double_integrator():
    """BASELINE configs[0]: DI, SVGD median, T=500, 100 iterations, eta=0.1."""
    g = load_golden("plan_cases.npz")
    q = fc.benchmark_mixture(2)
    res = fc.plan(fc.double_integrator_2d(), q, fc.Discretization(0.05, 500, DI_S0),
                  fc.PlanConfig(method="stein", eta=0.1, max_iterations=100,
                                convergence_tol=0.0, metric_interval=25, metric_samples=1000))
    assert res.iterations_used == 100
    assert rel_inf(res.trajectory.S, g["cfg1_S"]) <= 0.01
    assert rel_inf(res.flow_norms, g["cfg1_flow_norms"]) <= 0.01
    assert res.metric_iterations == tuple(int(v) for v in g["cfg1_metric_it"])
    assert res.final_metric == pytest.approx(float(g["cfg1_final_metric"]), rel=0.01)
    # per-iteration flows on identical inputs (the reference's own states)
    for i in range(3):
        X = g[f"cfg1_rec{i}_X"]
        a = fc.stein_flow(X, q).a
        assert rel_inf(a, g[f"cfg1_rec{i}_a"]) <= 1e-4


def test_config2_shape_sinkhorn_per_iteration_flows():
    """BASELINE configs[1] shape (T=2000, M=1e4): flows on the reference's states."""
    g = load_golden("plan_cases.npz")
    q = fc.benchmark_mixture(2)
    targets = fc.SamplePoints(q.sample(10_000, [0, STREAM_REFERENCE]))
    warm = fc.SinkhornWarmState()
    for i in range(3):
        a = fc.sinkhorn_flow(g[f"cfg2s_rec{i}_X"], targets, fc.SinkhornConfig(), warm=warm).a
        assert rel_inf(a, g[f"cfg2s_rec{i}_a"]) <= 1e-4, i
    res = fc.plan(fc.double_integrator_2d(), targets, fc.Discretization(0.05, 2000, DI_S0),
                  fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=3,
                                convergence_tol=0.0, metric_interval=0))
    assert rel_inf(res.trajectory.S, g["cfg2s_S"]) <= 0.01
    assert rel_inf(res.flow_norms, g["cfg2s_flow_norms"]) <= 1e-3


@pytest.mark.parametrize("tag,model,method,eta,iters,T,interval,samples,seed", [
    ("si_sk", "single_integrator_2d", "sinkhorn", 30.0, 20, 200, 5, 300, 0),
    ("dd_st", "diff_drive", "stein", 0.1, 15, 300, 5, 300, 4),
    ("ac_sk", "aircraft_3d", "sinkhorn", 45.0, 10, 300, 0, None, 0),
])
def test_small_plans_golden(tag, model, method, eta, iters, T, interval, samples, seed):
    g = load_golden("plan_cases.npz")
    m = fc.get_model(model)
    q = fc.benchmark_mixture(m.workspace_dim)
    res = fc.plan(m, q, fc.Discretization(0.05, T, fc.default_start(m)),
                  fc.PlanConfig(method=method, eta=eta, max_iterations=iters, convergence_tol=0.0,
                                metric_interval=interval, metric_samples=samples, seed=seed))
    assert rel_inf(res.trajectory.S, g[f"{tag}_S"]) <= 0.01
    assert rel_inf(res.trajectory.U, g[f"{tag}_U"]) <= 0.01
    assert rel_inf(res.lqr_costs, g[f"{tag}_lqr_costs"]) <= 0.01
    assert res.metric_iterations == tuple(int(v) for v in g[f"{tag}_metric_it"])
    if interval:
        np.testing.assert_allclose(res.metric_values, g[f"{tag}_metric_val"], rtol=0.01)


def test_config2_full_run_coverage():
    """200 outer iterations of BASELINE configs[1]: final coverage within 1%."""
    g = load_golden("plan_cfg2_full.npz")
    q = fc.benchmark_mixture(2)
    targets = fc.SamplePoints(q.sample(10_000, [0, STREAM_REFERENCE]))
    res = fc.plan(fc.double_integrator_2d(), targets, fc.Discretization(0.05, 2000, DI_S0),
                  fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=200,
                                convergence_tol=0.0, metric_interval=0))
    draws = q.sample(10_000, [0, STREAM_METRIC])
    cov = fc.coverage_metric(res.trajectory.S, fc.double_integrator_2d(), draws)
    assert cov == pytest.approx(float(g["cfg2_coverage"]), rel=0.01)
    assert rel_inf(res.trajectory.S, g["cfg2_S"]) <= 0.01


def test_converges_immediately_on_own_rollout():  # test_optimizer.py:32-43
    model = fc.single_integrator_2d()
    disc = fc.Discretization(dt=0.05, num_steps=50, s0=np.array([0.1, 0.1]))
    cfg = fc.PlanConfig(method="sinkhorn", seed=9, metric_interval=0)
    U0 = fc.initial_controls(cfg, model, disc.num_steps)
    S0 = fc.rollout(model, disc.s0, U0, disc.dt)
    res = fc.plan(model, fc.SamplePoints(points=S0[1:].copy()), disc, cfg)
    assert res.converged and res.iterations_used == 1
    assert res.flow_norms[0] < cfg.convergence_tol


def test_metric_cadence():  # test_optimizer.py:84-101
    model = fc.single_integrator_2d()
    disc = fc.Discretization(dt=0.05, num_steps=40, s0=np.array([0.1, 0.1]))
    cfg = fc.PlanConfig(method="stein", seed=1, max_iterations=12, convergence_tol=1e-12,
                        metric_interval=5, metric_samples=200)
    res = fc.plan(model, fc.benchmark_mixture(2), disc, cfg)
    assert not res.converged and res.iterations_used == 12
    assert res.metric_iterations == (0, 5, 10, 12)
    assert res.final_metric == res.metric_values[-1]
    assert len(res.flow_norms) == 12 and len(res.lqr_costs) == 12
    pt = res.phase_times
    assert pt.flow > 0 and pt.lqr > 0 and pt.rollout > 0
    assert pt.flow + pt.lqr + pt.rollout <= pt.total


def test_zero_start_clamped_reaches_target():  # test_optimizer.py:46-81
    model = fc.single_integrator_2d()
    q = fc.GaussianMixture(np.array([1.0]), np.array([[0.5, 0.5]]), (0.05 * np.eye(2))[None])
    disc = fc.Discretization(dt=0.05, num_steps=200, s0=np.array([0.1, 0.1]))
    cfg = fc.PlanConfig(method="stein", initial_controls="zeros", eta=0.1,
                        control_clamp=(1.0, 1.0), max_iterations=300, metric_interval=0)
    res = fc.plan(model, q, disc, cfg)
    targets = q.sample(2000, [0, STREAM_METRIC])
    final = fc.coverage_metric(res.trajectory.S, model, targets)
    initial = fc.coverage_metric(fc.rollout(model, disc.s0, np.zeros((200, 2)), disc.dt), model,
                                 targets)
    assert final < 0.2 * initial
    np.testing.assert_array_equal(res.trajectory.S,
                                  fc.rollout(model, disc.s0, res.trajectory.U, disc.dt))
    assert np.abs(res.trajectory.U).max() <= 1.0


def test_rollout_blowup_is_plan_error_with_context():  # test_optimizer.py:190-210
    model = fc.single_integrator_2d()
    disc = fc.Discretization(dt=0.05, num_steps=50, s0=np.array([0.1, 0.1]))
    cfg = fc.PlanConfig(method="stein", initial_controls="zeros", eta=1e308, max_iterations=5,
                        metric_interval=0)
    with pytest.raises(fc.PlanError) as exc:
        fc.plan(model, fc.benchmark_mixture(2), disc, cfg)
    err = exc.value
    assert err.stage == "rollout" and err.iteration == 1
    assert err.trajectory is not None and err.trajectory.S.shape == (51, 2)


def test_api_validation():  # test_optimizer.py:159-187
    model = fc.single_integrator_2d()
    disc = fc.Discretization(dt=0.05, num_steps=20, s0=np.zeros(2))
    with pytest.raises(ValueError, match="score-based"):
        fc.plan(model, fc.SamplePoints(np.random.default_rng(0).random((10, 2))), disc,
                fc.PlanConfig(method="stein"))
    dd = fc.differential_drive()
    with pytest.raises(ValueError, match="s0"):
        fc.plan(dd, fc.benchmark_mixture(2), fc.Discretization(0.05, 20, np.zeros(2)),
                fc.PlanConfig(metric_interval=0))
    with pytest.raises(ValueError, match="control_clamp"):
        fc.plan(dd, fc.benchmark_mixture(2), fc.Discretization(0.05, 20, np.zeros(3)),
                fc.PlanConfig(control_clamp=(1.0, 1.0, 1.0), metric_interval=0))
    res = fc.plan(model, fc.benchmark_mixture(2), fc.Discretization(0.05, 30, np.array([0.1, 0.1])),
                  fc.PlanConfig(method="sinkhorn", seed=3, max_iterations=3, metric_interval=0))
    assert res.iterations_used >= 1


def test_plan_is_run_to_run_deterministic():
    model = fc.differential_drive()
    disc = fc.Discretization(0.05, 120, np.array([0.1, 0.1, 0.0]))
    cfg = fc.PlanConfig(method="stein", seed=4, max_iterations=15, metric_interval=5,
                        metric_samples=300)
    a = fc.plan(model, fc.benchmark_mixture(2), disc, cfg)
    b = fc.plan(model, fc.benchmark_mixture(2), disc, cfg)
    assert a.trajectory.S.tobytes() == b.trajectory.S.tobytes()
    assert a.metric_values == b.metric_values


def test_plan_with_nvtx_ranges(monkeypatch):
    """FCB_NVTX=1 wraps the planner phases in NVTX ranges (ncu --nvtx
    filtering); results are unchanged."""
    from paper_2511_11514_b200 import _dev
    model = fc.single_integrator_2d()
    cfg = fc.PlanConfig(method="sinkhorn", eta=60.0, max_iterations=3, convergence_tol=0.0,
                        metric_interval=0)
    disc = fc.Discretization(0.05, 200, np.array([0.1, 0.1]))
    tg = fc.SamplePoints(fc.benchmark_mixture(2).sample(500, [0, 2]))
    a = fc.plan(model, tg, disc, cfg)
    monkeypatch.setattr(_dev, "NVTX", True)
    b = fc.plan(model, tg, disc, cfg)
    np.testing.assert_array_equal(a.trajectory.S, b.trajectory.S)
