"""Entropic optimal transport, the debiased divergence and its descent flow.

Drop-in for the reference's sinkhorn.py (sinkhorn.py:65-400) with the same
public names, signatures, error types and warm-start semantics.  Every solve
runs as one cooperative persistent kernel (`fcb_ot_solve`): the cost matrix
C = |x_i - y_j|^2 is evaluated tile by tile in registers and never stored,
the LSE sweeps are online max/sum-exp reductions, and the transport gradient
is taken from plan row masses and barycentres accumulated in the last sweep
(no T x M plan, no C^T copy).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import numpy.typing as npt
import torch

from . import _dev, _lib, _precision
from .flows import FlowField
from .parallel import resolve_workers
from .reference import SamplePoints

AUTO_OMEGA_FACTOR = 0.05
_OMEGA_FLOOR = 1e-12
_EXP_CLIP = 500.0


class SinkhornInputError(ValueError):
    """Inputs produced a cost matrix with non-finite entries."""


class FlowError(RuntimeError):
    """Transport solution too far from its marginals to trust the gradient."""


@dataclass(frozen=True)
class SinkhornConfig:
    """omega: "auto" (0.05 x mean squared X-Y distance) or a positive number.

    precision ("auto" | "float32" | "float64") selects the pairwise-kernel
    arithmetic; see _precision.py.  parallel_chunk / workers are validated
    but do not change results (the CUDA grid replaces the thread pool).
    """

    omega: float | str = "auto"
    max_iters: int = 1000
    tol: float = 1e-6
    parallel_chunk: int = 256
    workers: int | None = None
    precision: str = "auto"

    def __post_init__(self) -> None:
        if isinstance(self.omega, str):
            if self.omega != "auto":
                raise ValueError(f'omega must be "auto" or a number, got {self.omega!r}')
        elif not self.omega > 0:
            raise ValueError(f"omega must be positive, got {self.omega}")
        if self.max_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        if not self.tol > 0:
            raise ValueError(f"tol must be positive, got {self.tol}")
        if self.parallel_chunk < 1:
            raise ValueError(f"parallel_chunk must be >= 1, got {self.parallel_chunk}")
        if self.workers is not None and self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        _precision.validate(self.precision)


class SinkhornWarmState:
    """Dual potentials carried between flow evaluations, kept on the device.

    `f` / `p` read back as numpy arrays (or None), and may be assigned, like
    the reference's attributes (sinkhorn.py:104-115).  A potential whose
    length does not match the next problem is ignored (silent reset).
    """

    __slots__ = ("_f", "_p", "_valid", "_n")

    def __init__(self) -> None:
        self._f: torch.Tensor | None = None
        self._p: torch.Tensor | None = None
        self._valid: torch.Tensor | None = None
        self._n = 0

    def _ensure(self, n: int) -> None:
        dev = _dev.require_cuda()
        if self._f is None or self._n != n or self._f.device != dev:
            old_f, old_p = self.f_host_if(n), self.p_host_if(n)
            self._f = _dev.zeros((n,), device=dev)
            self._p = _dev.zeros((n,), device=dev)
            self._valid = torch.zeros(2, dtype=torch.int32, device=dev)
            self._n = n
            if old_f is not None:
                self._f.copy_(torch.from_numpy(old_f))
                self._valid[0] = 1
            if old_p is not None:
                self._p.copy_(torch.from_numpy(old_p))
                self._valid[1] = 1

    def f_host_if(self, n: int):
        f = self.f
        return f if f is not None and f.shape[0] == n else None

    def p_host_if(self, n: int):
        p = self.p
        return p if p is not None and p.shape[0] == n else None

    @property
    def f(self) -> np.ndarray | None:
        if self._f is None or int(self._valid[0]) == 0:
            return None
        return _dev.host(self._f).copy()

    @f.setter
    def f(self, value) -> None:
        self._set(0, value)

    @property
    def p(self) -> np.ndarray | None:
        if self._p is None or int(self._valid[1]) == 0:
            return None
        return _dev.host(self._p).copy()

    @p.setter
    def p(self, value) -> None:
        self._set(1, value)

    def _set(self, which: int, value) -> None:
        if value is None:
            if self._valid is not None:
                self._valid[which] = 0
            return
        arr = np.asarray(value, dtype=np.float64).ravel()
        other = self.p if which == 0 else self.f
        dev = _dev.require_cuda()
        n = arr.shape[0]
        if self._f is None or self._n != n:
            self._f = _dev.zeros((n,), device=dev)
            self._p = _dev.zeros((n,), device=dev)
            self._valid = torch.zeros(2, dtype=torch.int32, device=dev)
            self._n = n
            if other is not None and other.shape[0] == n:
                (self._p if which == 0 else self._f).copy_(torch.from_numpy(other))
                self._valid[1 - which] = 1
        (self._f if which == 0 else self._p).copy_(torch.from_numpy(arr))
        self._valid[which] = 1

    def device_buffers(self, n: int):
        """(f, p, valid) device tensors sized for n points (planner use)."""
        self._ensure(n)
        return self._f, self._p, self._valid


def _as_points(P, name: str) -> np.ndarray:
    P = np.atleast_2d(np.asarray(P, dtype=np.float64))
    if P.shape[0] < 1:
        raise SinkhornInputError(f"{name} must contain at least one point")
    if not np.isfinite(P).all():
        raise SinkhornInputError(f"{name} contains non-finite entries")
    return P


def _check_cost_finite(X: np.ndarray, Y: np.ndarray) -> None:
    """Raise like the reference when some |x_i - y_j|^2 overflows (sinkhorn.py:277-279).

    Summing the largest gap of each coordinate gives an upper bound on every
    C_ij in O(n + m).  For d > 1 those gaps can come from different pairs, so
    an overflowing bound is only a hint: the exact max_ij C_ij (row blocks, no
    (n, m) matrix) decides, as the reference's `np.isfinite(C).all()` does.
    """
    gap = np.maximum(X.max(axis=0) - Y.min(axis=0), Y.max(axis=0) - X.min(axis=0))
    with np.errstate(over="ignore", invalid="ignore"):
        bound = float((gap * gap).sum())
        if math.isfinite(bound):
            return
        step = max(1, (1 << 22) // max(Y.shape[0], 1))
        for lo in range(0, X.shape[0], step):
            blk = X[lo:lo + step]
            C = np.square(blk[:, :1] - Y[:, 0][None, :])
            for k in range(1, X.shape[1]):
                C += np.square(blk[:, k:k + 1] - Y[:, k][None, :])
            if not np.isfinite(C).all():
                raise SinkhornInputError("cost matrix has non-finite entries")


def _dims(X: np.ndarray, Y: np.ndarray) -> None:
    if X.shape[1] != Y.shape[1]:
        raise SinkhornInputError(f"point dims disagree: {X.shape[1]} vs {Y.shape[1]}")
    if X.shape[1] > 3:
        raise NotImplementedError("device kernels support workspaces of dimension 1-3")


def _omega_arg(omega) -> float:
    return 0.0 if isinstance(omega, str) else float(omega)


def _resolve_on_device(mode: int, prec: int, Xd, n, Yd, m, d, omega_fixed: float):
    scal = _dev.empty((16,))
    ws = _dev.Workspace.get(_lib.load().fcb_omega_workspace_bytes(n, m), "omega")
    _lib.call(
        "fcb_resolve_omega", mode | (prec << 8), _dev.ptr(Xd), n, _dev.ptr(Yd), m, d,
        omega_fixed, _dev.ptr(scal), _dev.ptr(ws), ws.numel(), _dev.stream(),
        what="resolve_omega", input_error=SinkhornInputError,
    )
    return scal


def resolve_omega(omega: float | str, X, Y) -> float:
    """Numeric omega; "auto" = max(0.05 mean_ij |x_i - y_j|^2, 1e-12) (sinkhorn.py:136-148)."""
    if not isinstance(omega, str):
        return float(omega)
    if omega != "auto":
        raise ValueError(f'omega must be "auto" or a number, got {omega!r}')
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    Y = np.atleast_2d(np.asarray(Y, dtype=np.float64))
    n, d = X.shape
    dev = _dev.require_cuda()
    Xd, Yd = _dev.f64(X, dev), _dev.f64(Y, dev)
    scal = _resolve_on_device(_lib.FCB_OT_ASYM, _lib.FCB_FP64, Xd, n, Yd, Y.shape[0], d, 0.0)
    return float(scal[0].item())


@dataclass(frozen=True)
class SinkhornSolution:
    """Dual solution of one transport problem (sinkhorn.py:239-256)."""

    f: npt.NDArray[np.float64]
    g: npt.NDArray[np.float64]
    cost: float
    iters_used: int
    converged: bool
    marginal_error: float
    omega: float
    X: npt.NDArray[np.float64]
    Y: npt.NDArray[np.float64]

    def plan(self) -> npt.NDArray[np.float64]:
        """Materialise the (n, m) plan exp((f_i + g_j - C_ij)/omega) on demand."""
        n, d = self.X.shape
        m = self.Y.shape[0]
        dev = _dev.require_cuda()
        Xd, Yd = _dev.f64(self.X, dev), _dev.f64(self.Y, dev)
        fd, gd = _dev.f64(self.f, dev), _dev.f64(self.g, dev)
        scal = _dev.zeros((16,), device=dev)
        scal[0] = self.omega
        out = _dev.empty((n, m), device=dev)
        _lib.call(
            "fcb_ot_plan", _dev.ptr(Xd), n, _dev.ptr(Yd), m, d, _dev.ptr(fd), _dev.ptr(gd),
            _dev.ptr(scal), _dev.ptr(out), _dev.stream(), what="ot_plan",
        )
        return _dev.host(out)


def entropic_ot(
    X,
    Y,
    cfg: SinkhornConfig = SinkhornConfig(),
    workers: int | None = None,
    omega: float | None = None,
    f0=None,
) -> SinkhornSolution:
    """Solve entropic OT between two point sets (sinkhorn.py:259-300)."""
    X = _as_points(X, "X")
    Y = _as_points(Y, "Y")
    _dims(X, Y)
    _check_cost_finite(X, Y)
    resolve_workers(workers or cfg.workers)
    n, d = X.shape
    m = Y.shape[0]
    prec = _precision.pick(cfg.precision, n * m, cfg.tol)
    dev = _dev.require_cuda()
    Xd, Yd = _dev.f64(X, dev), _dev.f64(Y, dev)
    fixed = float(omega) if omega is not None else _omega_arg(cfg.omega)
    scal = _resolve_on_device(_lib.FCB_OT_ASYM, prec, Xd, n, Yd, m, d, fixed)
    f0d = None
    if f0 is not None:
        f0 = np.asarray(f0, dtype=np.float64).ravel()
        if f0.shape[0] != n:
            raise ValueError(f"f0 must have {n} entries, got {f0.shape[0]}")
        f0d = _dev.f64(f0, dev)
    f, g, rs = _dev.empty((n,)), _dev.empty((m,)), _dev.empty((n,))
    stat, cost = _dev.empty((4,)), _dev.empty((1,))
    lib = _lib.load()
    ws = _dev.Workspace.get(lib.fcb_ot_workspace_bytes(_lib.FCB_OT_ASYM, prec, n, m, d), "ot")
    _lib.call(
        "fcb_ot_solve", _lib.FCB_OT_ASYM, prec, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d,
        _dev.ptr(scal), cfg.max_iters, cfg.tol, _dev.ptr(f0d), _dev.ptr(f), _dev.ptr(g),
        _dev.ptr(rs), _dev.ptr(stat), None, None, _dev.ptr(ws), ws.numel(), _dev.stream(),
        what="entropic_ot", input_error=SinkhornInputError,
    )
    _lib.call(
        "fcb_ot_cost", _lib.FCB_OT_ASYM, _dev.ptr(f), _dev.ptr(rs), n, _dev.ptr(g), m,
        _dev.ptr(cost), _dev.stream(), what="ot_cost",
    )
    st = _dev.host(stat)
    return SinkhornSolution(
        f=_dev.host(f),
        g=_dev.host(g),
        cost=float(cost.item()),
        iters_used=int(st[1]),
        converged=bool(st[2] != 0.0),
        marginal_error=float(st[0]),
        omega=float(scal[0].item()),
        X=X,
        Y=Y,
    )


def sinkhorn_divergence(
    X,
    Y,
    cfg: SinkhornConfig = SinkhornConfig(),
    workers: int | None = None,
) -> float:
    """Debiased S_w(X, Y) = OT(X,Y) - (OT(X,X) + OT(Y,Y))/2, one shared omega."""
    X = _as_points(X, "X")
    Y = _as_points(Y, "Y")
    _dims(X, Y)
    _check_cost_finite(X, Y)
    resolve_workers(workers or cfg.workers)
    n, d = X.shape
    m = Y.shape[0]
    prec = _precision.pick(cfg.precision, max(n, m) ** 2, cfg.tol)
    dev = _dev.require_cuda()
    Xd, Yd = _dev.f64(X, dev), _dev.f64(Y, dev)
    out = _dev.empty((4,))
    lib = _lib.load()
    ws = _dev.Workspace.get(lib.fcb_sinkhorn_divergence_workspace_bytes(prec, n, m, d), "div")
    _lib.call(
        "fcb_sinkhorn_divergence", prec, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d,
        _omega_arg(cfg.omega), cfg.max_iters, cfg.tol, _dev.ptr(out), None, _dev.ptr(ws),
        ws.numel(), _dev.stream(), what="sinkhorn_divergence", input_error=SinkhornInputError,
    )
    return float(out[0].item())


def lse_sweep(X, Y, pot, omega: float, precision: str = "float32") -> np.ndarray:
    """One _lse_rows sweep (sinkhorn.py:151-167): out_i = LSE_j((pot_j - |x_i - y_j|^2)/omega).

    The primitive every solve iterates; exposed for parity tests and the
    roofline measurement in bench.py.
    """
    X = _as_points(X, "X")
    Y = _as_points(Y, "Y")
    _dims(X, Y)
    n, d = X.shape
    m = Y.shape[0]
    prec = _precision.pick(precision, n * m)
    dev = _dev.require_cuda()
    Xd, Yd, potd = _dev.f64(X, dev), _dev.f64(Y, dev), _dev.f64(np.ravel(pot), dev)
    scal = _resolve_on_device(_lib.FCB_OT_SWEEP, prec, Xd, n, Yd, m, d, float(omega))
    out = _dev.empty((n,))
    lib = _lib.load()
    ws = _dev.Workspace.get(lib.fcb_ot_workspace_bytes(_lib.FCB_OT_SWEEP, prec, n, m, d), "ot")
    _lib.call(
        "fcb_ot_solve", _lib.FCB_OT_SWEEP, prec, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d,
        _dev.ptr(scal), 1, 0.0, _dev.ptr(potd), _dev.ptr(out), None, None, None, None, None,
        _dev.ptr(ws), ws.numel(), _dev.stream(), what="lse_sweep",
    )
    return _dev.host(out)


def flow_error_message(worst: float, tol: float) -> str:
    return (
        f"transport marginals violated by {worst:.3e} (> 100 * tol = {100 * tol:.3e}); "
        "increase max_iters or omega"
    )


def sinkhorn_flow(
    X,
    q: SamplePoints,
    cfg: SinkhornConfig = SinkhornConfig(),
    workers: int | None = None,
    warm: SinkhornWarmState | None = None,
    *,
    stats: dict | None = None,
) -> FlowField:
    """Minus the divergence gradient at each point of X (sinkhorn.py:338-400).

    stats (additive, keyword-only): receives omega and the inner iteration
    counts of the cross and self solves (iters_cross, iters_self).
    """
    X = _as_points(X, "X")
    Y = _as_points(q.points, "reference points")
    _dims(X, Y)
    _check_cost_finite(X, Y)
    resolve_workers(workers or cfg.workers)
    n, d = X.shape
    m = Y.shape[0]
    prec = _precision.pick(cfg.precision, n * max(n, m), cfg.tol)
    dev = _dev.require_cuda()
    Xd, Yd = _dev.f64(X, dev), _dev.f64(Y, dev)
    flow, fstat = _dev.empty((n, d)), _dev.empty((8,))
    wf = wp = wv = None
    if warm is not None:
        wf, wp, wv = warm.device_buffers(n)
    lib = _lib.load()
    ws = _dev.Workspace.get(lib.fcb_sinkhorn_flow_workspace_bytes(prec, n, m, d), "flow")
    _lib.call(
        "fcb_sinkhorn_flow", prec, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d, _omega_arg(cfg.omega),
        cfg.max_iters, cfg.tol, _dev.ptr(wf), _dev.ptr(wp), _dev.ptr(wv), _dev.ptr(flow),
        _dev.ptr(fstat), None, 0, None, 0.0, _dev.ptr(ws), ws.numel(), _dev.stream(),
        what="sinkhorn_flow", input_error=SinkhornInputError,
    )
    st = _dev.host(fstat)
    worst = float(st[0])
    if stats is not None:
        stats.update(omega=float(st[4]), iters_cross=int(st[5]), iters_self=int(st[6]),
                     worst=worst)
    if st[2] != 0.0:
        raise FlowError(flow_error_message(worst, cfg.tol))
    return FlowField(a=_dev.host(flow), converged=bool(st[1] != 0.0), marginal_error=worst)
