"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/flowcover_oracle.py) is the parity checker for the CUDA
path at sizes beyond the fixtures; these tests show it reproduces the
reference's outputs (bit-for-bit where the arithmetic is identical).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import flowcover_oracle as O
from fcb_testutil import load_golden, rel_inf


def _omega(cfg):
    return "auto" if cfg[0] == 0.0 else float(cfg[0])


def test_entropic_ot_matches_reference():
    g = load_golden("ot_cases.npz")
    for k in range(int(g["ncases"])):
        X, Y, cfg = g[f"c{k}_X"], g[f"c{k}_Y"], g[f"c{k}_cfg"]
        r = O.entropic_ot(X, Y, _omega(cfg), int(cfg[1]), float(cfg[2]))
        scal = g[f"c{k}_scal"]
        assert np.array_equal(r["f"], g[f"c{k}_f"]), k
        assert np.array_equal(r["g"], g[f"c{k}_g"]), k
        assert r["iters"] == int(scal[1]) and r["converged"] == bool(scal[2])
        assert r["cost"] == pytest.approx(scal[0], rel=1e-14, abs=1e-300)
        assert r["omega"] == scal[4]


def test_single_lse_sweep_bit_identical():
    g = load_golden("ot_cases.npz")
    L = O.lse_sweep(g["sweep_X"], g["sweep_Y"], g["sweep_pot"], float(g["sweep_omega"]))
    assert np.array_equal(L, g["sweep_L"])


def test_sweep_independent_of_chunk_and_workers():
    g = load_golden("ot_cases.npz")
    X, Y, pot = g["sweep_X"][:700], g["sweep_Y"], g["sweep_pot"]
    a = O.lse_sweep(X, Y, pot, 0.02, chunk=256, workers=1)
    b = O.lse_sweep(X, Y, pot, 0.02, chunk=37, workers=4)
    assert np.array_equal(a, b)


def test_sinkhorn_flow_and_warm_start_match_reference():
    g = load_golden("flow_cases.npz")
    for k in range(int(g["ncases"])):
        X, Y, cfg = g[f"c{k}_X"], g[f"c{k}_Y"], g[f"c{k}_cfg"]
        if X.shape[0] * Y.shape[0] > 2_000_000:
            continue  # the big case is checked on the GPU only
        warm: dict = {}
        a, conv, err = O.sinkhorn_flow(X, Y, _omega(cfg), int(cfg[1]), float(cfg[2]), warm)
        assert np.array_equal(a, g[f"c{k}_a"]), k
        a2, _, _ = O.sinkhorn_flow(g[f"c{k}_X2"], Y, _omega(cfg), int(cfg[1]), float(cfg[2]), warm)
        assert np.array_equal(a2, g[f"c{k}_a2"]), k
        assert np.array_equal(warm["f"], g[f"c{k}_warm_f"])
        if f"c{k}_div" in g:
            d = O.sinkhorn_divergence(X, Y, _omega(cfg), int(cfg[1]), float(cfg[2]))
            assert d == pytest.approx(float(g[f"c{k}_div"]), rel=1e-12, abs=1e-15)


def test_stein_and_median_match_reference():
    g = load_golden("stein_cases.npz")
    for k in range(int(g["ncases"])):
        X, dim, bw = g[f"c{k}_X"], int(g[f"c{k}_dim"]), float(g[f"c{k}_bw"])
        if dim == 1:
            q = O.Mixture([1.0], np.zeros((1, 1)), np.eye(1)[None])
        else:
            q = O.benchmark_mixture(dim)
        a, h, _ = O.stein_flow(X, q, "median" if bw < 0 else bw)
        assert h == float(g[f"c{k}_h"])
        assert rel_inf(a, g[f"c{k}_a"]) <= 1e-13, k
        assert O.median_bandwidth(X) == float(g[f"c{k}_med_h"])


def test_mixture_score_density_and_sampling_match_reference():
    g = load_golden("stein_cases.npz")
    q = O.Mixture(g["gmm_w"], g["gmm_mu"], g["gmm_cov"])
    assert rel_inf(q.score(g["gmm_X"]), g["gmm_score"]) <= 1e-13
    assert rel_inf(q.log_density(g["gmm_X"]), g["gmm_logd"]) <= 1e-14
    q3 = O.benchmark_mixture(3)
    assert rel_inf(q3.score(g["gmm3_X"]), g["gmm3_score"]) <= 1e-13
    assert np.array_equal(O.benchmark_mixture(2).sample(1000, [0, 3]), g["sample2"])


@pytest.mark.parametrize("name", ["single_integrator_2d", "diff_drive", "aircraft_3d",
                                  "double_integrator_2d"])
def test_rollout_and_linearization_match_reference(name):
    g = load_golden("dyn_lqr_cases.npz")
    f, ja, jb, _ = O.model_fns(name)
    S, fail = O.rollout(f, g[f"{name}_s0"], g[f"{name}_U"], 0.05)
    assert fail == -1
    assert np.array_equal(S, g[f"{name}_S"])
    A, B = O.linearize(ja, jb, S, g[f"{name}_U"])
    assert np.array_equal(A, g[f"{name}_A"]) and np.array_equal(B, g[f"{name}_B"])


@pytest.mark.parametrize("T", [1, 2, 3, 5, 10, 200, 2000])
def test_lqr_matches_reference(T):
    g = load_golden("dyn_lqr_cases.npz")
    p = f"lqr{T}_"
    r = O.solve_flow_lqr(g[p + "A"], g[p + "B"], 0.05, g[p + "a"], g[p + "Q"], g[p + "R"])
    assert rel_inf(r["v"], g[p + "v"]) <= 1e-12
    assert rel_inf(r["z"], g[p + "z"]) <= 1e-12
    assert r["cost"] == pytest.approx(float(g[p + "cost"]), rel=1e-12)


def test_plan_loop_matches_reference_short_runs():
    g = load_golden("plan_cases.npz")
    # aircraft + sinkhorn, 10 iterations
    q3 = O.benchmark_mixture(3)
    r = O.plan("aircraft_3d", np.array([0.1, 0.1, 0.35, 0.0, 0.0, 0.2]), 0.05, 300, "sinkhorn",
               45.0, 10, q=q3, seed=0)
    assert rel_inf(r["S"], g["ac_sk_S"]) <= 1e-10
    assert rel_inf(r["flow_norms"], g["ac_sk_flow_norms"]) <= 1e-10
    # single integrator + sinkhorn, 20 iterations
    r = O.plan("single_integrator_2d", np.array([0.1, 0.1]), 0.05, 200, "sinkhorn", 30.0, 20,
               q=O.benchmark_mixture(2), seed=0)
    assert rel_inf(r["S"], g["si_sk_S"]) <= 1e-10
    assert rel_inf(r["lqr_costs"], g["si_sk_lqr_costs"]) <= 1e-10
