"""Multi-GPU execution of the flow: M-sharded Sinkhorn and batched problems.

One process per GPU (torch.distributed, NCCL over NVLink on a B200 box).

M-sharded Sinkhorn flow (BASELINE config 4).  Rank r holds a
shard Y_r of the reference samples; X and the potentials f (and p) are
replicated.  One inner iteration of _solve_asymmetric (sinkhorn.py:170-205):

    g_r   = w (log b - LSE_rows(Y_r vs X, f))        local, log b = -log M
    L_r   = LSE_rows(X vs Y_r, g_r)                   local partial (n,)
    L     = LSE over ranks of L_r                     one all_gather of n doubles,
                                                      merged in fixed rank order
    f_new = w (log a - L); err from f and f_new       replicated -> identical
                                                      branch on every rank

The transport gradient needs sum_j T_ij y_j over all shards: every f-sweep
also returns the per-shard barycentre, combined with the same softmax weights
exp(L_r - L).  The self term OT(X, X) involves no reference samples and is
solved redundantly (identically) on every rank.  omega "auto" uses the
global mean statistics of Y (one all_reduce).

The sweep itself is pluggable: on a GPU it is the fp32/fp64 sweep of
fcb_ot_solve(FCB_OT_SWEEP); tests/ inject the CPU oracle to check the
collective logic with the gloo backend on CPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _dev, _lib, _precision
from .flows import FlowField
from .sinkhorn import (
    AUTO_OMEGA_FACTOR,
    FlowError,
    SinkhornConfig,
    _EXP_CLIP,
    _OMEGA_FLOOR,
    _resolve_on_device,
    flow_error_message,
)

# sweep(R, S, pot, omega, with_bary) -> (L (rows,), bary (rows, d) or None),
# L_i = LSE_j((pot_j - |r_i - s_j|^2) / omega) in natural units.
SweepFn = Callable[[torch.Tensor, torch.Tensor, torch.Tensor, float, bool], tuple]


def cuda_sweep(precision: str = "auto") -> SweepFn:
    """The device sweep (fcb_ot_solve in FCB_OT_SWEEP mode)."""

    def sweep(R, S, pot, omega, with_bary):
        n, d = R.shape
        m = S.shape[0]
        prec = _precision.pick(precision, n * m)
        scal = _resolve_on_device(_lib.FCB_OT_SWEEP, prec, R, n, S, m, d, float(omega))
        out = _dev.empty((n,), device=R.device)
        bary = _dev.empty((n, d + 1), device=R.device) if with_bary else None
        lib = _lib.load()
        ws = _dev.Workspace.get(lib.fcb_ot_workspace_bytes(_lib.FCB_OT_SWEEP, prec, n, m, d), "dist")
        potc = pot.contiguous()
        _lib.call(
            "fcb_ot_solve", _lib.FCB_OT_SWEEP, prec, _dev.ptr(R), n, _dev.ptr(S), m, d,
            _dev.ptr(scal), 1, 0.0, _dev.ptr(potc), _dev.ptr(out), None, None, None,
            _dev.ptr(bary), None, _dev.ptr(ws), ws.numel(), _dev.stream(), what="sweep",
        )
        return out, (bary[:, 1:] if with_bary else None)

    return sweep


def _world(group) -> tuple[int, int]:
    if group is None or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _all_gather(t: torch.Tensor, group) -> list[torch.Tensor]:
    rank, world = _world(group)
    if world == 1:
        return [t]
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous(), group=group)
    return parts


def _all_reduce_sum(t: torch.Tensor, group) -> torch.Tensor:
    _, world = _world(group)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def lse_merge(parts: list[torch.Tensor]) -> tuple[torch.Tensor, list[torch.Tensor]]:
    """log-sum-exp over shards, fixed order; also the per-shard weights exp(L_r - L)."""
    stacked = torch.stack(parts)  # (R, n)
    top = stacked.max(dim=0).values
    top = torch.where(torch.isfinite(top), top, torch.zeros_like(top))
    w = torch.exp(stacked - top)
    total = w.sum(dim=0)
    L = top + torch.log(total)
    weights = [w[r] / total for r in range(len(parts))]
    return L, weights


def global_omega(omega, X: torch.Tensor, Y_local: torch.Tensor, group) -> float:
    """resolve_omega (sinkhorn.py:136-148) with Y statistics reduced over ranks."""
    if not isinstance(omega, str):
        return float(omega)
    d = X.shape[1]
    stats = torch.zeros(d + 2, dtype=torch.float64, device=Y_local.device)
    stats[:d] = Y_local.sum(dim=0)
    stats[d] = (Y_local * Y_local).sum()
    stats[d + 1] = float(Y_local.shape[0])
    _all_reduce_sum(stats, group)
    m = stats[d + 1]
    ybar = stats[:d] / m
    y2 = stats[d] / m
    xbar = X.mean(dim=0)
    x2 = (X * X).sum(dim=1).mean()
    mean_sq = float(x2 + y2 - 2.0 * (xbar @ ybar))
    return max(AUTO_OMEGA_FACTOR * mean_sq, _OMEGA_FLOOR)


@dataclass
class ShardedSolution:
    f: torch.Tensor
    g_local: torch.Tensor
    row_sums: torch.Tensor
    row_mass: torch.Tensor  # unclipped plan row sums
    ybar: torch.Tensor  # global plan barycentres (n, d)
    err: float
    iters: int
    converged: bool


def sharded_asymmetric(X, Y_local, omega, max_iters, tol, f0, m_global, sweep: SweepFn,
                       group=None) -> ShardedSolution:
    """_solve_asymmetric (sinkhorn.py:170-205) with Y sharded over `group`."""
    n = X.shape[0]
    loga, logb = -math.log(n), -math.log(m_global)
    f = torch.zeros(n, dtype=torch.float64, device=X.device) if f0 is None else f0.clone()
    it = 0
    while True:
        it += 1
        Lg, _ = sweep(Y_local, X, f, omega, False)
        g = omega * (logb - Lg)
        L_r, ybar_r = sweep(X, Y_local, g, omega, True)
        parts = _all_gather(L_r, group)
        bparts = _all_gather(ybar_r, group)
        L, weights = lse_merge(parts)
        ybar = sum(w[:, None] * b for w, b in zip(weights, bparts))
        f_new = omega * (loga - L)
        delta = torch.clamp((f - f_new) / omega, max=_EXP_CLIP)  # NaN propagates
        err = float(torch.abs(torch.expm1(delta)).max()) / n
        if err <= tol or it >= max_iters:
            return ShardedSolution(
                f=f, g_local=g, row_sums=torch.exp(delta + loga),
                row_mass=torch.exp(f / omega + L), ybar=ybar, err=err, iters=it,
                converged=err <= tol,
            )
        f = f_new


def replicated_symmetric(X, omega, max_iters, tol, p0, sweep: SweepFn):
    """_solve_symmetric (sinkhorn.py:208-236), identical on every rank."""
    n = X.shape[0]
    loga = -math.log(n)
    p = torch.zeros(n, dtype=torch.float64, device=X.device) if p0 is None else p0.clone()
    it = 0
    while True:
        it += 1
        L, xbar = sweep(X, X, p, omega, True)
        target = omega * (loga - L)
        delta = torch.clamp((p - target) / omega, max=_EXP_CLIP)
        err = float(torch.abs(torch.expm1(delta)).max()) / n
        if err <= tol or it >= max_iters:
            return p, torch.exp(delta + loga), torch.exp(p / omega + L), xbar, err, it, err <= tol
        p = 0.5 * (p + target)


class ShardedSinkhornFlow:
    """sinkhorn_flow (sinkhorn.py:338-400) over reference samples sharded across ranks.

    Keeps the warm potentials (f, p) between calls like SinkhornWarmState.
    """

    def __init__(self, Y_local, cfg: SinkhornConfig = SinkhornConfig(), group=None,
                 sweep: Optional[SweepFn] = None, device=None):
        self.group = group
        self.cfg = cfg
        self.device = device or (_dev.require_cuda() if sweep is None else torch.device("cpu"))
        self.Y = torch.as_tensor(np.asarray(Y_local, dtype=np.float64)).to(self.device)
        self.sweep = sweep or cuda_sweep(cfg.precision)
        m = torch.tensor([float(self.Y.shape[0])], dtype=torch.float64, device=self.device)
        self.m_global = int(_all_reduce_sum(m, group).item())
        self.f = None
        self.p = None

    def __call__(self, X) -> FlowField:
        X = torch.as_tensor(np.asarray(X, dtype=np.float64)).to(self.device)
        n = X.shape[0]
        cfg = self.cfg
        w = global_omega(cfg.omega, X, self.Y, self.group)
        f0 = self.f if self.f is not None and self.f.shape[0] == n else None
        p0 = self.p if self.p is not None and self.p.shape[0] == n else None
        cross = sharded_asymmetric(X, self.Y, w, cfg.max_iters, cfg.tol, f0, self.m_global,
                                   self.sweep, self.group)
        p, rho, rho_u, xbar, err_p, _, conv_p = replicated_symmetric(
            X, w, cfg.max_iters, cfg.tol, p0, self.sweep)
        worst = max(cross.err, err_p)
        if worst > 100.0 * cfg.tol:
            raise FlowError(flow_error_message(worst, cfg.tol))
        grad = (2.0 * (cross.row_sums[:, None] * X - cross.row_mass[:, None] * cross.ybar)
                - 2.0 * (rho[:, None] * X - rho_u[:, None] * xbar))
        self.f, self.p = cross.f, p
        return FlowField(a=(-grad).cpu().numpy(), converged=cross.converged and conv_p,
                         marginal_error=worst)


def shard_rows(Y: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Contiguous, balanced shard `rank` of the rows of Y."""
    m = Y.shape[0]
    lo = (m * rank) // world
    hi = (m * (rank + 1)) // world
    return Y[lo:hi]


def plan_batch(problems: list, group=None) -> list:
    """Independent planning problems split across ranks (BASELINE config 5).

    problems: list of (model, q, disc, cfg).  Rank r plans problems r, r+R,
    ...; results are gathered on every rank in problem order.  No collective
    touches the data path.
    """
    from .optimizer import plan_batch as plan_local

    rank, world = _world(group)
    idx = list(range(rank, len(problems), world))
    mine = dict(zip(idx, plan_local([problems[i] for i in idx])))
    if world == 1:
        return [mine[i] for i in range(len(problems))]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    out = {}
    for part in gathered:
        out.update(part)
    return [out[i] for i in range(len(problems))]
