"""Rollout, linearisation and the flow-matching LQR on the GPU."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2511_11514_b200 as fc
from fcb_testutil import load_golden, rel_inf

pytestmark = pytest.mark.gpu

MODELS = {
    "single_integrator_2d": fc.single_integrator_2d,
    "diff_drive": fc.differential_drive,
    "aircraft_3d": fc.aircraft_3d,
    "double_integrator_2d": fc.double_integrator_2d,
}


@pytest.mark.parametrize("name", sorted(MODELS))
def test_rollout_and_linearization_golden(name):
    g = load_golden("dyn_lqr_cases.npz")
    m = MODELS[name]()
    S = fc.rollout(m, g[f"{name}_s0"], g[f"{name}_U"], 0.05)
    if name in ("single_integrator_2d", "double_integrator_2d"):
        assert np.array_equal(S, g[f"{name}_S"])  # polynomial models: bit-exact
    else:
        assert rel_inf(S, g[f"{name}_S"]) <= 1e-12
    sys_ = fc.linearize_along(m, g[f"{name}_S"], g[f"{name}_U"], 0.05)
    assert rel_inf(sys_.A, g[f"{name}_A"]) <= 1e-13
    assert rel_inf(sys_.B, g[f"{name}_B"]) <= 1e-13


def test_rollout_kats():  # test_dynamics.py:117-160
    m = fc.single_integrator_2d()
    S = fc.rollout(m, np.zeros(2), np.tile([1.0, 0.0], (10, 1)), 0.1)
    np.testing.assert_allclose(S[10], [1.0, 0.0], atol=1e-12)
    dd = fc.differential_drive()
    S = fc.rollout(dd, np.zeros(3), np.tile([1.0, 0.0], (10, 1)), 0.1)
    np.testing.assert_allclose(S[10], [1.0, 0.0, 0.0], atol=1e-12)

    def arc_error(steps):
        dt = np.pi / steps
        S = fc.rollout(dd, np.zeros(3), np.tile([1.0, 1.0], (steps, 1)), dt)
        t = dt * np.arange(steps + 1)
        return np.abs(S - np.column_stack([np.sin(t), 1.0 - np.cos(t), t])).max()

    assert arc_error(50) <= 1e-6
    assert arc_error(50) / arc_error(100) >= 8.0
    with pytest.raises(fc.RolloutDivergenceError) as exc:
        fc.rollout(m, np.zeros(2), np.full((5, 2), 1e308), 0.1)
    assert exc.value.step == 1


def test_lti_user_model_rollout():
    A = np.array([[0.0, 1.0], [-1.0, -0.1]])
    B = np.array([[0.0], [1.0]])
    lin = fc.DynamicsModel(
        name="osc", state_dim=2, control_dim=1, workspace_dim=1, state_names=("x", "v"),
        control_names=("a",), f=lambda s, u: A @ s + B @ u, jacobian_A=lambda s, u: A.copy(),
        jacobian_B=lambda s, u: B.copy(), project_matrix=np.array([[1.0, 0.0]]),
    )
    from oracle import flowcover_oracle as O

    U = np.random.default_rng(0).normal(size=(100, 1))
    S = fc.rollout(lin, np.array([1.0, 0.0]), U, 0.05)
    ref, _ = O.rollout(lin.f, np.array([1.0, 0.0]), U, 0.05)
    assert rel_inf(S, ref) <= 1e-14


@pytest.mark.parametrize("T", [1, 2, 3, 5, 10, 200, 2000])
def test_lqr_golden(T):
    g = load_golden("dyn_lqr_cases.npz")
    p = f"lqr{T}_"
    sol = fc.solve_flow_lqr(fc.LtvSystem(A=g[p + "A"], B=g[p + "B"], dt=0.05), g[p + "a"],
                            fc.LqrWeights(Q=g[p + "Q"], R=g[p + "R"]))
    assert rel_inf(sol.v_star, g[p + "v"]) <= 1e-10
    assert rel_inf(sol.z, g[p + "z"]) <= 1e-10
    assert rel_inf(sol.K, g[p + "K"]) <= 1e-10
    assert sol.cost == pytest.approx(float(g[p + "cost"]), rel=1e-10)


@pytest.mark.parametrize("T,n,m", [(4096, 4, 2), (4097, 4, 2), (2049, 6, 3), (12000, 3, 2)])
def test_lqr_long_horizon_matches_oracle(T, n, m):
    """Both affine-phase paths: the single-CTA fused scan (T <= 8 * block) and
    the three-kernel multi-CTA scan above it."""
    from oracle import flowcover_oracle as O

    rng = np.random.default_rng(T + n)
    A = 0.2 * rng.normal(size=(T, n, n)) - 0.5 * np.eye(n)
    B = rng.normal(size=(T, n, m))
    Q, R = np.eye(n), 0.1 * np.eye(m)
    a = np.cumsum(rng.normal(scale=0.1, size=(T, n)), axis=0)
    sol = fc.solve_flow_lqr(fc.LtvSystem(A=A, B=B, dt=0.05), a, fc.LqrWeights(Q=Q, R=R))
    ref = O.solve_flow_lqr(A, B, 0.05, a, Q, R)
    assert rel_inf(sol.v_star, ref["v"]) <= 1e-9
    assert rel_inf(sol.z, ref["z"]) <= 1e-9
    assert sol.cost == pytest.approx(ref["cost"], rel=1e-9)


def dense_solution(A, B, dt, a, Q, R):  # the normal-equation oracle of test_lqr.py:44-63
    T, n, _ = A.shape
    m = B.shape[2]
    maps, M = [], np.zeros((n, T * m))
    for k in range(T):
        maps.append(M.copy())
        M = (np.eye(n) + dt * A[k]) @ M
        M[:, k * m:(k + 1) * m] += dt * B[k]
    H, b = np.zeros((T * m, T * m)), np.zeros(T * m)
    for k in range(T):
        H += dt * maps[k].T @ Q @ maps[k]
        b += dt * maps[k].T @ (Q @ a[k])
        H[k * m:(k + 1) * m, k * m:(k + 1) * m] += dt * R
    return np.linalg.solve(H, b).reshape(T, m)


@pytest.mark.parametrize("T", [1, 2, 3, 5, 10])
def test_lqr_matches_dense_quadratic(T):
    rng = np.random.default_rng(100 + T)
    A, B = 0.3 * rng.normal(size=(T, 3, 3)), rng.normal(size=(T, 3, 2))
    C, D = rng.normal(size=(3, 3)), rng.normal(size=(2, 2))
    Q, R = C.T @ C, D.T @ D + 0.1 * np.eye(2)
    a = rng.normal(size=(T, 3))
    sol = fc.solve_flow_lqr(fc.LtvSystem(A=A, B=B, dt=0.05), a, fc.LqrWeights(Q=Q, R=R))
    assert np.abs(sol.v_star - dense_solution(A, B, 0.05, a, Q, R)).max() <= 1e-8


def test_lqr_kats():  # test_lqr.py:69-96, 195-208
    rng = np.random.default_rng(0)
    sys_ = fc.LtvSystem(A=0.3 * rng.normal(size=(12, 3, 3)), B=rng.normal(size=(12, 3, 2)), dt=0.05)
    w = fc.LqrWeights(Q=np.eye(3), R=0.1 * np.eye(2))
    sol = fc.solve_flow_lqr(sys_, np.zeros((12, 3)), w)
    assert np.array_equal(sol.v_star, np.zeros((12, 2))) and sol.cost == 0.0
    one = fc.solve_flow_lqr(fc.LtvSystem(A=np.zeros((1, 2, 2)), B=np.eye(2)[None], dt=0.1),
                            np.array([[5.0, -3.0]]), fc.LqrWeights(Q=np.eye(2), R=0.1 * np.eye(2)))
    assert np.array_equal(one.v_star, np.zeros((1, 2)))
    dt = 0.1
    two = fc.solve_flow_lqr(fc.LtvSystem(A=np.zeros((2, 1, 1)), B=np.ones((2, 1, 1)), dt=dt),
                            np.array([[0.0], [1.0]]), fc.LqrWeights(Q=np.eye(1), R=0.1 * np.eye(1)))
    assert two.v_star[0, 0] == pytest.approx(2 * dt / (0.2 + 2 * dt * dt), abs=1e-12)
    assert two.v_star[1, 0] == 0.0
    T = 300
    blow = fc.LtvSystem(A=np.tile(1e306 * np.eye(2), (T, 1, 1)), B=np.tile(np.eye(2), (T, 1, 1)),
                        dt=0.05)
    with pytest.raises(fc.RiccatiDivergenceError) as exc:
        fc.solve_flow_lqr(blow, np.ones((T, 2)), fc.LqrWeights(Q=np.eye(2), R=0.1 * np.eye(2)))
    assert 0 <= exc.value.step < T
