"""Helpers shared by the test modules (fixtures, tolerances)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name: str) -> dict:
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing (run tests/golden/make_golden.py)")
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def rel_inf(a, b) -> float:
    """max|a-b| / max|b|: the north_star's infinity-norm relative error."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))
