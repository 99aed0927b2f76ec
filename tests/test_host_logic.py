"""Host-side logic that needs no GPU: configs, validation, model resolution."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2511_11514_b200 as fc
from paper_2511_11514_b200 import _lib, _precision
from paper_2511_11514_b200.dynamics import device_model
from paper_2511_11514_b200.parallel import chunk_ranges, resolve_workers


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        fc.PlanConfig(eta=0.0)
    with pytest.raises(ValueError):
        fc.PlanConfig(max_iterations=0)
    with pytest.raises(ValueError):
        fc.PlanConfig(method="gradient")
    with pytest.raises(ValueError):
        fc.PlanConfig(initial_controls="tiny")
    with pytest.raises(ValueError):
        fc.SinkhornConfig(omega="medium")
    with pytest.raises(ValueError):
        fc.SinkhornConfig(omega=-1.0)
    with pytest.raises(ValueError):
        fc.SinkhornConfig(precision="half")
    with pytest.raises(ValueError):
        fc.SteinConfig(bandwidth=0.0)
    assert fc.PlanConfig(control_clamp=[1, 2]).control_clamp == (1.0, 2.0)


def test_precision_auto_rule():
    assert _precision.pick("auto", 10**8, 1e-6) == _lib.FCB_FP32
    assert _precision.pick("auto", 10**8, 1e-10) == _lib.FCB_FP64
    assert _precision.pick("auto", 1000, 1e-6) == _lib.FCB_FP64
    assert _precision.pick("float32", 10, 1e-12) == _lib.FCB_FP32


def test_mixture_validation_and_sampling_streams():
    with pytest.raises(ValueError, match="sum to 1"):
        fc.GaussianMixture(np.array([0.5, 0.4]), np.zeros((2, 2)), np.stack([np.eye(2)] * 2))
    with pytest.raises(ValueError, match="positive definite"):
        fc.GaussianMixture(np.array([1.0]), np.zeros((1, 2)), np.array([[[1.0, 2.0], [2.0, 1.0]]]))
    q = fc.benchmark_mixture(2)
    assert np.array_equal(q.sample(5, 7), q.sample(5, 7))
    sb = fc.to_sample_based(q, 10, 3)
    assert np.array_equal(sb.points, q.sample(10, 3))
    with pytest.raises(ValueError):
        fc.SamplePoints(points=np.array([[0.0, np.inf]]))


def test_sampling_is_bit_identical_to_the_oracle():
    from oracle import flowcover_oracle as O

    assert np.array_equal(fc.benchmark_mixture(3).sample(777, [0, 2]),
                          O.benchmark_mixture(3).sample(777, [0, 2]))


def test_device_model_resolution():
    assert device_model(fc.single_integrator_2d()).model_id == _lib.FCB_MODEL_SINGLE_INTEGRATOR_2D
    assert device_model(fc.differential_drive()).model_id == _lib.FCB_MODEL_DIFF_DRIVE
    assert device_model(fc.aircraft_3d()).model_id == _lib.FCB_MODEL_AIRCRAFT_3D
    assert device_model(fc.double_integrator_2d()).model_id == _lib.FCB_MODEL_DOUBLE_INTEGRATOR_2D
    # a user-built linear model becomes the generic LTI device model
    A = np.array([[0.0, 1.0], [-1.0, -0.1]])
    B = np.array([[0.0], [1.0]])
    lin = fc.DynamicsModel(
        name="my_oscillator", state_dim=2, control_dim=1, workspace_dim=1,
        state_names=("x", "v"), control_names=("a",),
        f=lambda s, u: A @ s + B @ u, jacobian_A=lambda s, u: A.copy(),
        jacobian_B=lambda s, u: B.copy(), project_matrix=np.array([[1.0, 0.0]]),
    )
    spec = device_model(lin)
    assert spec.model_id == _lib.FCB_MODEL_LTI
    assert np.array_equal(spec.params, np.concatenate([A.ravel(), B.ravel()]))
    # a nonlinear model with no device twin is refused, not run on the CPU
    pend = fc.DynamicsModel(
        name="pendulum", state_dim=2, control_dim=1, workspace_dim=1,
        state_names=("th", "om"), control_names=("tau",),
        f=lambda s, u: np.array([s[1], -np.sin(s[0]) + u[0]]),
        jacobian_A=lambda s, u: np.array([[0.0, 1.0], [-np.cos(s[0]), 0.0]]),
        jacobian_B=lambda s, u: np.array([[0.0], [1.0]]),
        project_matrix=np.array([[1.0, 0.0]]),
    )
    with pytest.raises(NotImplementedError):
        device_model(pend)
    # a model named like a device model but behaving differently is not trusted
    fake = fc.DynamicsModel(
        name="single_integrator_2d", state_dim=2, control_dim=2, workspace_dim=2,
        state_names=("x", "y"), control_names=("a", "b"),
        f=lambda s, u: 2.0 * np.asarray(u), jacobian_A=lambda s, u: np.zeros((2, 2)),
        jacobian_B=lambda s, u: 2.0 * np.eye(2), project_matrix=np.eye(2),
    )
    assert device_model(fake).model_id == _lib.FCB_MODEL_LTI


def test_workers_knobs_validate_like_reference(monkeypatch):
    assert resolve_workers(3) == 3
    monkeypatch.setenv("FLOWCOVER_WORKERS", "5")
    assert resolve_workers() == 5
    monkeypatch.setenv("FLOWCOVER_WORKERS", "x")
    with pytest.raises(ValueError):
        resolve_workers()
    assert chunk_ranges(5, 2) == [(0, 2), (2, 4), (4, 5)]


def test_lqr_weights_and_lift():
    m = fc.differential_drive()
    w = fc.workspace_weights(m.project_matrix, m.control_dim, q_weight=2.0, r_weight=0.3)
    np.testing.assert_allclose(w.Q, np.diag([2.0, 2.0, 0.0]))
    np.testing.assert_allclose(fc.lift_flow(np.array([[1.0, 2.0]]), m.project_matrix), [[1.0, 2.0, 0.0]])
    with pytest.raises(ValueError):
        fc.LqrWeights(Q=np.array([[1.0, 0.0], [0.0, -1.0]]), R=np.eye(2))


def test_compute_entry_points_fail_loudly_without_a_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeLibraryError):
        fc.sinkhorn_flow(np.random.rand(5, 2), fc.SamplePoints(np.random.rand(6, 2)))
    with pytest.raises(_lib.NativeLibraryError):
        fc.rollout(fc.single_integrator_2d(), np.zeros(2), np.ones((3, 2)), 0.1)


def test_bench_plugin_planners_build_without_gpu():
    """bench_plugin mirrors the reference harness's planner closures (bench.py:158-209)."""
    from types import SimpleNamespace

    from paper_2511_11514_b200 import bench_plugin

    spec = SimpleNamespace(model="diff_drive", dt=0.05, seed=3, plan=None)
    planners = bench_plugin.b200_planners(spec)
    assert set(planners) == {"b200-stein", "b200-sinkhorn"}
    assert all(callable(p) for p in planners.values())
    assert bench_plugin.STUDY_ITERATIONS == 20 and bench_plugin.STUDY_BANDWIDTH == 0.02


def test_cost_finite_check_uses_exact_pairs():
    """sinkhorn.py:277-279 raises only when some C_ij itself overflows."""
    from paper_2511_11514_b200.sinkhorn import SinkhornInputError, _check_cost_finite

    # per-coordinate gaps overflow together, but no single pair does
    _check_cost_finite(np.array([[1.2e154, 0.0], [0.0, 1.2e154]]), np.zeros((1, 2)))
    with pytest.raises(SinkhornInputError):
        _check_cost_finite(np.array([[1.2e154, 1.2e154]]), np.zeros((1, 2)))
    with pytest.raises(SinkhornInputError):
        _check_cost_finite(np.array([[1e200]]), np.array([[-1e200]]))
