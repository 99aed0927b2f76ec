"""Tours of the TSP-waypoint baseline on the GPU (reference tsp.py:76-147) vs
tours the unmodified reference built (tests/golden/make_golden_r2.py): the same
move sequence means the same order, bit for bit, and the same length."""

from __future__ import annotations

import numpy as np
import pytest

from fcb_testutil import load_golden
from paper_2511_11514_b200 import tsp

pytestmark = pytest.mark.gpu
TAGS = ["t0", "t1", "t3d", "tbud", "t2", "tdup"]


@pytest.mark.parametrize("tag", TAGS)
def test_tour_matches_reference(tag):
    g = load_golden("tsp_cases.npz")
    seed, budget, length = g[f"{tag}_meta"]
    tour = tsp.build_tour(g[f"{tag}_pts"], int(seed), None if budget < 0 else int(budget))
    np.testing.assert_array_equal(tour.order, g[f"{tag}_order"])
    assert tour.length == length


def test_batched_tours_match_single_ones():
    g = load_golden("tsp_cases.npz")
    probs = [(g["t0_pts"], 0, None), (g["t1_pts"], 1, None), (g["t0_pts"], 5, None)]
    tours = tsp.build_tours(probs)
    np.testing.assert_array_equal(tours[0].order, g["t0_order"])
    np.testing.assert_array_equal(tours[1].order, g["t1_order"])
    np.testing.assert_array_equal(tours[2].order, tsp.build_tour(g["t0_pts"], 5).order)


def test_tour_input_validation():
    with pytest.raises(ValueError):
        tsp.build_tour(np.zeros((1, 2)), 0)
    with pytest.raises(ValueError):
        tsp.build_tours([(np.zeros((3, 2)), 0, None), (np.zeros((4, 2)), 1, None)])


# ---- tracking stage and the whole baseline (tsp.py:150-316) ----------------
def _rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("tag,model,d", [("si", "single_integrator_2d", 2),
                                         ("dd", "diff_drive", 2), ("ac", "aircraft_3d", 3)])
def test_baseline_plan_matches_reference(tag, model, d):
    """Targets and tour bit-identical; the tracked trajectory (10 rounds of
    device linearise / Riccati / affine update) within 1e-8 of the reference's
    float64 numpy."""
    import paper_2511_11514_b200 as fc
    g = load_golden("track_cases.npz")
    seed, T = (int(v) for v in g[f"{tag}_meta"])
    m = fc.get_model(model)
    res = fc.baseline_plan(m, fc.benchmark_mixture(d), fc.Discretization(0.05, T, fc.default_start(m)),
                           fc.BaselineConfig(seed=seed))
    np.testing.assert_array_equal(res.waypoints, g[f"{tag}_waypoints"])
    np.testing.assert_array_equal(res.tour.order, g[f"{tag}_order"])
    assert _rel(res.trajectory.S, g[f"{tag}_S"]) <= 1e-8
    assert _rel(res.trajectory.U, g[f"{tag}_U"]) <= 1e-8
    pt = res.phase_times
    assert pt.lqr > 0 and pt.rollout > 0 and pt.total >= pt.flow


def test_track_waypoints_repeated_points_and_errors():
    import paper_2511_11514_b200 as fc
    g = load_golden("track_cases.npz")
    S, U = fc.track_waypoints(fc.differential_drive(), g["rep_W"], 120, 0.05, iterations=6)
    assert _rel(S, g["rep_S"]) <= 1e-8 and _rel(U, g["rep_U"]) <= 1e-8
    with pytest.raises(ValueError):
        fc.track_waypoints(fc.differential_drive(), g["rep_W"][:1], 10, 0.05)
    with pytest.raises(ValueError):
        fc.track_waypoints(fc.differential_drive(), g["rep_W"], 0, 0.05)
    with pytest.raises(ValueError, match="no reference lift"):
        fc.track_waypoints(fc.double_integrator_2d(), g["rep_W"], 10, 0.05)


def test_batched_baselines_equal_single_ones():
    import paper_2511_11514_b200 as fc
    m = fc.single_integrator_2d()
    q = fc.benchmark_mixture(2)
    disc = fc.Discretization(0.05, 200, np.array([0.1, 0.1]))
    cfgs = [fc.BaselineConfig(seed=s) for s in (3, 4)] + [fc.BaselineConfig(seed=5, budget=50)]
    many = fc.baseline_plans(m, q, disc, cfgs)
    for c, r in zip(cfgs, many):
        one = fc.baseline_plan(m, q, disc, c)
        np.testing.assert_array_equal(r.tour.order, one.tour.order)
        np.testing.assert_array_equal(r.trajectory.S, one.trajectory.S)
        np.testing.assert_array_equal(r.trajectory.U, one.trajectory.U)
