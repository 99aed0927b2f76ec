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
