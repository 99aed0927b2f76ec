"""Stein flow, median bandwidth and mixture score on the GPU.

Known-answer tests follow the reference's test_stein.py / test_reference.py;
golden parity uses vectors produced by the reference.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2511_11514_b200 as fc
from fcb_testutil import load_golden, rel_inf
from oracle import flowcover_oracle as O

pytestmark = pytest.mark.gpu


def standard_normal(dim=2):
    return fc.GaussianMixture(np.array([1.0]), np.zeros((1, dim)), np.eye(dim)[None])


def test_stein_golden_and_exact_median():
    g = load_golden("stein_cases.npz")
    for k in range(int(g["ncases"])):
        X, dim, bw = g[f"c{k}_X"], int(g[f"c{k}_dim"]), float(g[f"c{k}_bw"])
        q = standard_normal(1) if dim == 1 else fc.benchmark_mixture(dim)
        # the median is selected exactly: bandwidths are bit-identical
        assert fc.median_bandwidth(X) == float(g[f"c{k}_med_h"]), k
        out = fc.stein_flow(X, q, fc.SteinConfig(bandwidth="median" if bw < 0 else bw))
        assert out.bandwidth == float(g[f"c{k}_h"])
        assert rel_inf(out.a, g[f"c{k}_a"]) <= 1e-4, (k, rel_inf(out.a, g[f"c{k}_a"]))


@pytest.mark.parametrize("n", [999, 1000, 2048, 4097])
def test_fp32_stein_vs_oracle(n):
    rng = np.random.default_rng(n)
    X = rng.random((n, 2))
    q = fc.benchmark_mixture(2)
    out = fc.stein_flow(X, q, fc.SteinConfig(bandwidth="median", precision="float32"))
    ref, h, _ = O.stein_flow(X, O.benchmark_mixture(2), "median")
    assert out.bandwidth == h
    assert rel_inf(out.a, ref) <= 1e-4


def test_mixture_score_and_density_golden():
    g = load_golden("stein_cases.npz")
    q = fc.GaussianMixture(g["gmm_w"], g["gmm_mu"], g["gmm_cov"])
    assert rel_inf(q.score(g["gmm_X"]), g["gmm_score"]) <= 1e-12
    assert rel_inf(q.log_density(g["gmm_X"]), g["gmm_logd"]) <= 1e-13
    q3 = fc.benchmark_mixture(3)
    assert rel_inf(q3.score(g["gmm3_X"]), g["gmm3_score"]) <= 1e-12
    assert rel_inf(q3.log_density(g["gmm3_X"]), g["gmm3_logd"]) <= 1e-13


def test_score_kats():  # test_reference.py:65-81
    q = standard_normal()
    assert np.array_equal(q.score(np.zeros((1, 2))), np.zeros((1, 2)))
    np.testing.assert_allclose(q.score(np.array([[2.0, 0.0]])), [[-2.0, 0.0]], atol=1e-12)
    q2 = fc.GaussianMixture(np.array([0.5, 0.5]), np.array([[1.0, 0.0], [-1.0, 0.0]]),
                            np.stack([0.25 * np.eye(2)] * 2))
    np.testing.assert_allclose(q2.score(np.zeros((1, 2))), [[0.0, 0.0]], atol=1e-12)


def test_single_point_kats():  # test_stein.py:31-40
    out = fc.stein_flow(np.zeros((1, 2)), standard_normal(), fc.SteinConfig(bandwidth=1.0))
    assert np.array_equal(out.a, np.zeros((1, 2)))
    out = fc.stein_flow(np.array([[2.0, 0.0]]), standard_normal(), fc.SteinConfig(bandwidth=1.0))
    np.testing.assert_allclose(out.a, [[-2.0, 0.0]], atol=1e-14)


def test_two_point_closed_form():  # test_stein.py:43-53
    pts = np.array([[1.0, 0.0], [-1.0, 0.0]])
    k12 = np.exp(-4.0)
    g1 = 0.5 * (-pts[0] + (-k12 * pts[1] + 2.0 * (pts[0] - pts[1]) * k12))
    g2 = 0.5 * (-pts[1] + (-k12 * pts[0] + 2.0 * (pts[1] - pts[0]) * k12))
    out = fc.stein_flow(pts, standard_normal(), fc.SteinConfig(bandwidth=1.0))
    np.testing.assert_allclose(out.a, [g1, g2], atol=1e-14)


def test_translation_and_permutation_equivariance():  # test_stein.py:56-67, 127-135
    rng = np.random.default_rng(11)
    pts = rng.normal(size=(15, 2))
    shift = rng.uniform(-5, 5, 2)
    q = standard_normal()
    qs = fc.GaussianMixture(q.weights, q.means + shift, q.covariances)
    base = fc.stein_flow(pts, q, fc.SteinConfig(bandwidth=0.7)).a
    moved = fc.stein_flow(pts + shift, qs, fc.SteinConfig(bandwidth=0.7)).a
    np.testing.assert_allclose(moved, base, atol=1e-12)
    pts = rng.normal(size=(40, 2))
    perm = rng.permutation(40)
    qb = fc.benchmark_mixture(2)
    a = fc.stein_flow(pts, qb, fc.SteinConfig(bandwidth=0.2)).a
    b = fc.stein_flow(pts[perm], qb, fc.SteinConfig(bandwidth=0.2)).a
    np.testing.assert_allclose(b, a[perm], rtol=1e-12, atol=1e-14)


def test_median_fallback_and_clamp():  # test_stein.py:79-91
    assert fc.median_bandwidth(np.array([[3.0, 1.0]])) == 1.0
    out = fc.stein_flow(np.array([[2.0, 0.0]]), standard_normal(), fc.SteinConfig())
    assert out.bandwidth == 1.0 and not out.clamped
    out = fc.stein_flow(np.tile([0.3, 0.4], (8, 1)), standard_normal(), fc.SteinConfig())
    assert out.clamped and out.bandwidth == 1e-12 and np.isfinite(out.a).all()


def test_median_matches_numpy_on_ties_and_odd_even():
    rng = np.random.default_rng(5)
    for n in (2, 3, 40, 41, 128):
        X = np.round(rng.random((n, 2)) * 4) / 4  # many tied distances
        assert fc.median_bandwidth(X) == O.median_bandwidth(X), n


def test_trajectory_flow_skips_start():  # test_stein.py:105-124
    m = fc.single_integrator_2d()
    rng = np.random.default_rng(2)
    U = rng.normal(scale=0.5, size=(30, 2))
    S = fc.rollout(m, np.array([0.1, 0.1]), U, 0.05)
    q = fc.benchmark_mixture(2)
    cfg = fc.SteinConfig(bandwidth=0.1)
    via = fc.stein_flow_on_trajectory(S, m, q, cfg)
    assert np.array_equal(via.a, fc.stein_flow(S[1:], q, cfg).a)
    assert via.num_steps == 30
    dd = fc.differential_drive()
    S = fc.rollout(dd, np.zeros(3), rng.normal(scale=0.5, size=(25, 2)), 0.05)
    assert fc.stein_flow_on_trajectory(S, dd, q).a.shape == (25, 2)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_median_cluster_and_cooperative_paths_exact(d):
    """Small sets take the one-cluster selection (keys in shared memory,
    histograms merged over DSMEM), larger ones the cooperative kernel; both
    select exactly numpy's median (bit-identical bandwidths)."""
    from paper_2511_11514_b200 import _lib
    rng = np.random.default_rng(40 + d)
    for n, want in ((500, "median_cluster_kernel"), (801, "median_cluster_kernel"),
                    (1500, "median_coop_kernel")):
        for ties in (False, True):
            X = rng.random((n, d))
            if ties:
                X = np.round(X * 6) / 6
            assert fc.median_bandwidth(X) == O.median_bandwidth(X), (n, d, ties)
            assert _lib.last_kernel() == want, (n, d, _lib.last_kernel())
