"""Tour construction of the TSP-waypoint baseline, on the GPU.

Drop-in for the tour half of the reference's tsp.py (tsp.py:30-147): the same
`Tour`, `tour_length` and `build_tour(points, seed, budget)` signatures and
results.  The nearest-neighbour order and the first-improving 2-opt search
run in `fcb_tsp_tours` (csrc/tsp.cu), one CTA per problem with the point set
in shared memory; `build_tours` plans many problems in one launch (BASELINE
config 5 compares 4096 planned problems against 4096 TSP baselines).  Only the
start index is drawn on the host, from the reference's stream [seed, 4].

The tour is the baseline the flow planners are compared with, not the
product; it lives here so the comparison can be run at config-5 scale.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import numpy.typing as npt
import torch

from . import _dev, _lib
from .seeding import STREAM_TOUR, rng_stream

IMPROVEMENT_EPS = 1e-12  # tsp.py:27 (the kernel uses the same margin)


@dataclass(frozen=True)
class Tour:
    """Open (non-returning) visiting order over a fixed point set."""

    order: npt.NDArray[np.int64]
    length: float

    def __post_init__(self) -> None:
        order = np.asarray(self.order, dtype=np.int64)
        object.__setattr__(self, "order", order)
        if order.ndim != 1 or not np.array_equal(np.sort(order), np.arange(order.size)):
            raise ValueError("order must be a permutation of 0..n-1")


def tour_length(points, order) -> float:
    """Length of the open path through points[order] (tsp.py:69-73)."""
    P = np.asarray(points, dtype=np.float64)[np.asarray(order)]
    if len(P) < 2:
        return 0.0
    return float(np.sqrt(((P[1:] - P[:-1]) ** 2).sum(axis=1)).sum())


def _check(points) -> np.ndarray:
    P = np.asarray(points, dtype=np.float64)
    if P.ndim != 2 or len(P) < 2:
        raise ValueError("need at least two points of equal dimension")
    return P


def build_tours(problems) -> list[Tour]:
    """build_tour of every (points, seed, budget) problem, one CTA each.

    All point sets must share n and d (budget may differ only through None /
    0 = automatic, i.e. 10 n).
    """
    sets = [_check(p) for p, _, _ in problems]
    if not sets:
        return []
    n, d = sets[0].shape
    if any(s.shape != (n, d) for s in sets):
        raise ValueError("batched tours need point sets of one shape")
    budgets = {(b if b else 10 * n) for _, _, b in problems}
    if len(budgets) != 1:
        raise ValueError("batched tours need one move budget")
    budget = budgets.pop()
    starts = np.array([int(rng_stream(seed, STREAM_TOUR).integers(n)) for _, seed, _ in problems],
                      dtype=np.int32)
    dev = _dev.require_cuda()
    pts = _dev.f64(np.stack(sets), dev)
    st = torch.from_numpy(starts).to(dev)
    B = len(sets)
    order = torch.empty((B, n), dtype=torch.int32, device=dev)
    moves = torch.empty(B, dtype=torch.int32, device=dev)
    _lib.call("fcb_tsp_tours", _dev.ptr(pts), B, n, d, _dev.ptr(st), int(budget), _dev.ptr(order),
              _dev.ptr(moves), _dev.stream(), what="tsp_tours")
    orders = order.cpu().numpy().astype(np.int64)
    return [Tour(order=o, length=tour_length(s, o)) for o, s in zip(orders, sets)]


def build_tour(points, seed: int, budget: int | None = None) -> Tour:
    """Nearest-neighbour tour from a seeded random start, refined by 2-opt
    (tsp.py:120-147); budget None / 0 means 10 n moves."""
    return build_tours([(points, seed, budget)])[0]
