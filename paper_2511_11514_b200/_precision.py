"""Arithmetic-precision selection for the pairwise kernels.

The pairwise LSE / kernel sweeps have a float32 instantiation (MUFU.EX2,
expanded form, the production path) and a float64 one (IEEE exp, direct
form).  float32 meets the north_star tolerance (1e-4 relative on flows and
potentials) at the default tol=1e-6, but it cannot
certify marginal errors far below ~1e-7 and the reference's own known-answer
tests use tol down to 1e-12.  "auto" therefore picks float64 for tight
tolerances and for small problems (< 2^20 pairs per sweep, where the sweep
is launch-latency bound and float64 costs nothing measurable), float32
otherwise.
"""

from __future__ import annotations

from . import _lib

PRECISIONS = ("auto", "float32", "float64")
SMALL_PAIRS = 1 << 20
TIGHT_TOL = 1e-7


def validate(p: str) -> None:
    if p not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}, got {p!r}")


def pick(p: str, pairs: int, tol: float | None = None) -> int:
    validate(p)
    if p == "float32":
        return _lib.FCB_FP32
    if p == "float64":
        return _lib.FCB_FP64
    if tol is not None and tol < TIGHT_TOL:
        return _lib.FCB_FP64
    return _lib.FCB_FP64 if pairs < SMALL_PAIRS else _lib.FCB_FP32
