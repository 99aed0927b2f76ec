"""The fused planner (one persistent launch for the coverage loop) against the
per-iteration device loop, and the batched many-problem path (BASELINE config
5) against per-problem plan() calls.

Both paths implement optimizer.py:221-269 with the same kernels' arithmetic;
they differ only in summation order (the fused LQR/rollout scans chunk the
time axis differently) -- results agree to fp64/fp32 rounding, far inside the
north_star's 1 % trajectory tolerance.  Reference parity of the loop itself is
tests/test_gpu_plan.py (config 2 golden run, which takes the fused path).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2511_11514_b200 as fc
from fcb_testutil import load_golden, rel_inf

pytestmark = pytest.mark.gpu
DI_S0 = np.array([0.1, 0.1, 0.0, 0.0])


def _plan(fused: bool, *args):
    old = os.environ.get("FCB_FUSED")
    os.environ["FCB_FUSED"] = "1" if fused else "0"
    try:
        return fc.plan_detailed(*args)
    finally:
        if old is None:
            os.environ.pop("FCB_FUSED")
        else:
            os.environ["FCB_FUSED"] = old


@pytest.mark.parametrize("model_name", ["double_integrator_2d", "single_integrator_2d"])
def test_fused_matches_per_iteration_loop(model_name):
    model = getattr(fc, model_name)()
    s0 = DI_S0 if model.state_dim == 4 else np.array([0.1, 0.1])
    q = fc.benchmark_mixture(2)
    Y = q.sample(3000, [0, 2])
    cfg = fc.PlanConfig(method="sinkhorn", eta=120.0, max_iterations=25, convergence_tol=0.0,
                        metric_interval=0)
    disc = fc.Discretization(0.05, 800, s0)
    a = _plan(True, model, fc.SamplePoints(Y), disc, cfg)
    b = _plan(False, model, fc.SamplePoints(Y), disc, cfg)
    ra, rb = a.result, b.result
    assert ra.iterations_used == rb.iterations_used == 25
    assert rel_inf(ra.trajectory.S, rb.trajectory.S) <= 1e-4
    assert rel_inf(ra.trajectory.U, rb.trajectory.U) <= 1e-4
    assert rel_inf(ra.flow_norms, rb.flow_norms) <= 1e-4
    assert rel_inf(ra.lqr_costs, rb.lqr_costs) <= 1e-4
    # inner iteration counts: the err-vs-tol test can flip by one iteration
    # when two paths' rounding differs (~1e-7) right at the threshold
    assert np.abs(a.flow_log[:, 1:3] - b.flow_log[:, 1:3]).max() <= 1
    assert abs(a.pairs - b.pairs) <= 0.01 * b.pairs
    assert ra.phase_times.flow > 0 and ra.phase_times.lqr > 0 and ra.phase_times.rollout > 0


def test_fused_stops_on_convergence():
    model = fc.double_integrator_2d()
    q = fc.benchmark_mixture(2)
    Y = q.sample(2000, [0, 2])
    disc = fc.Discretization(0.05, 600, DI_S0)
    cfg = fc.PlanConfig(method="sinkhorn", eta=90.0, max_iterations=60, convergence_tol=5e-3,
                        metric_interval=0)
    a = _plan(True, model, fc.SamplePoints(Y), disc, cfg).result
    b = _plan(False, model, fc.SamplePoints(Y), disc, cfg).result
    assert a.converged == b.converged
    assert a.iterations_used == b.iterations_used
    assert len(a.lqr_costs) == len(b.lqr_costs)
    assert rel_inf(a.trajectory.S, b.trajectory.S) <= 1e-4


def test_fused_config2_golden():
    """BASELINE configs[1] end to end (fused path) vs the reference's golden run."""
    g = load_golden("plan_cfg2_full.npz")
    q = fc.benchmark_mixture(2)
    Y = q.sample(10_000, [0, 2])
    res = _plan(True, fc.double_integrator_2d(), fc.SamplePoints(Y),
                fc.Discretization(0.05, 2000, DI_S0),
                fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=200,
                              convergence_tol=0.0, metric_interval=0)).result
    assert res.iterations_used == 200
    assert rel_inf(res.trajectory.S, g["cfg2_S"]) <= 0.01
    assert rel_inf(res.flow_norms, g["cfg2_flow_norms"]) <= 0.01


@pytest.mark.parametrize("model_name", ["single_integrator_2d", "double_integrator_2d"])
def test_batched_problems_match_individual_plans(model_name):
    """Config-5 shape (independent problems, seed b per problem), reduced."""
    model = getattr(fc, model_name)()
    q = fc.benchmark_mixture(2)
    T, M, B = 400, 1024, 5
    problems = []
    for b in range(B):
        s0 = np.zeros(model.state_dim)
        s0[:2] = (0.1 + 0.05 * b, 0.1)
        problems.append((model, fc.SamplePoints(q.sample(M, [b, 2])),
                         fc.Discretization(0.05, T, s0),
                         fc.PlanConfig(method="sinkhorn", eta=60.0, max_iterations=12,
                                       convergence_tol=0.0, metric_interval=0, seed=b)))
    batched = fc.plan_batch_detailed(problems)
    assert len(batched) == B
    for b, (m, qq, ds, c) in enumerate(problems):
        ref = _plan(False, m, qq, ds, c)
        got = batched[b]
        assert got.result.iterations_used == ref.result.iterations_used == 12
        assert rel_inf(got.result.trajectory.S, ref.result.trajectory.S) <= 1e-4
        assert rel_inf(got.result.flow_norms, ref.result.flow_norms) <= 1e-4
        assert rel_inf(got.result.lqr_costs, ref.result.lqr_costs) <= 1e-4
        assert np.abs(got.flow_log[:, 1:3] - ref.flow_log[:, 1:3]).max() <= 1


def test_bench_plugin_runs_planners():
    from types import SimpleNamespace

    from paper_2511_11514_b200 import bench_plugin

    spec = SimpleNamespace(model="single_integrator_2d", dt=0.05, seed=0, plan=None)
    planners = bench_plugin.b200_planners(spec)
    for name in ("b200-stein", "b200-sinkhorn"):
        run = planners[name](60, 1)
        assert run.trajectory.S.shape == (61, 2)
        assert run.t_flow > 0 and run.t_lqr >= 0 and run.t_rollout > 0


# ---- the fused SVGD planner (sv_plan_kernel) --------------------------------
@pytest.mark.parametrize("model_name,bw", [("double_integrator_2d", "median"),
                                           ("single_integrator_2d", "median"),
                                           ("double_integrator_2d", 0.02)])
def test_fused_stein_matches_per_iteration_loop(model_name, bw):
    """Rollout, score, exact median, fp64 Stein flow and LQR update in one
    launch vs the per-iteration kernels: the same fp64 arithmetic up to
    summation order, so trajectories, flow norms, bandwidths and costs agree
    to ~1e-10."""
    from paper_2511_11514_b200 import _lib
    model = getattr(fc, model_name)()
    s0 = DI_S0 if model.state_dim == 4 else np.array([0.1, 0.1])
    cfg = fc.PlanConfig(method="stein", eta=0.1, max_iterations=30, convergence_tol=0.0,
                        metric_interval=0, stein=fc.SteinConfig(bandwidth=bw))
    disc = fc.Discretization(0.05, 500, s0)
    a = _plan(True, model, fc.benchmark_mixture(2), disc, cfg)
    assert "sv_plan_kernel" in _lib.last_kernel() or a.launches < 30 * 4
    b = _plan(False, model, fc.benchmark_mixture(2), disc, cfg)
    ra, rb = a.result, b.result
    assert ra.iterations_used == rb.iterations_used == 30
    assert rel_inf(ra.trajectory.S, rb.trajectory.S) <= 1e-9
    assert rel_inf(ra.trajectory.U, rb.trajectory.U) <= 1e-9
    assert rel_inf(ra.flow_norms, rb.flow_norms) <= 1e-9
    assert rel_inf(ra.lqr_costs, rb.lqr_costs) <= 1e-9
    # the bandwidth column of the flow log: the median is exact on both paths
    assert rel_inf(a.flow_log[:, 1], b.flow_log[:, 1]) <= 1e-9
    assert ra.phase_times.flow > 0 and ra.phase_times.lqr > 0 and ra.phase_times.rollout > 0


def test_fused_stein_stops_on_convergence():
    model = fc.double_integrator_2d()
    disc = fc.Discretization(0.05, 400, DI_S0)
    cfg = fc.PlanConfig(method="stein", eta=0.1, max_iterations=80, convergence_tol=2e-2,
                        metric_interval=0)
    a = _plan(True, model, fc.benchmark_mixture(2), disc, cfg).result
    b = _plan(False, model, fc.benchmark_mixture(2), disc, cfg).result
    assert a.converged == b.converged
    assert a.iterations_used == b.iterations_used
    assert len(a.lqr_costs) == len(b.lqr_costs)
    assert rel_inf(a.trajectory.S, b.trajectory.S) <= 1e-9

