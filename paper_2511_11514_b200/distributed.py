"""Multi-GPU execution of the flows: M-sharded Sinkhorn, source-sharded SVGD,
batched independent problems.

One process per GPU (torch.distributed, NCCL over NVLink on a B200 box).  This
replaces the reference's only parallelism, the row-chunked thread pool of
parallel.py:47-66 used by sinkhorn.py:151-167 and stein.py:110-121.

M-sharded Sinkhorn flow (BASELINE config 4).  Rank r holds a
contiguous shard Y_r of the reference samples; X, f and p are replicated.
One inner iteration of _solve_asymmetric (sinkhorn.py:170-205):

    g_r   = w (log b - LSE_rows(Y_r vs X; f))      local sweep, log b = -log M
    {L_r, ybar_r} = LSE_rows(X vs Y_r; g_r)        local sweep + barycentres
    all_gather {L_r, ybar_r}                        n (d+1) doubles per rank
    f_new = w (log a - LSE_r L_r), err              fixed rank order -> every
                                                    rank holds identical f and
                                                    takes the same branch

The self term OT(X, X) (_solve_symmetric, sinkhorn.py:208-236) is row-sharded:
rank r sweeps its rows of X against all of X, and the updated rows of p (with
their plan masses, barycentres and errors) are all-gathered each iteration.
omega "auto" uses the global Y statistics (one all_reduce per planner call).

Every step is a device kernel (csrc/shard.cu) or an NCCL collective on the
same stream; loop control is a device word per solve, the host only queues
iterations ahead and polls completed snapshots (no per-iteration round trip).

SVGD (stein.py:79-122) shards the sources j: each rank sums k_ij and
k_ij (s_j - (2/h) x_j) over its sources for all queries; the partials are
all-gathered and summed in rank order.

The device steps sit behind an `ops` object (DeviceOps: the C ABI).  tests/
substitute a CPU implementation of the same steps to run the collective
schedule with the gloo backend and world sizes 2 and 4.
"""

from __future__ import annotations

import collections
import math
import os
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _dev, _lib, _precision
from .flows import FlowField
from .sinkhorn import FlowError, SinkhornConfig, _omega_arg, flow_error_message


def _world(group) -> tuple[int, int]:
    if group is None or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard [lo, hi) of n rows (csrc/shard.cu shard_of_row)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def shard_rows(Y: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Contiguous, balanced shard `rank` of the rows of Y."""
    lo, hi = shard_bounds(Y.shape[0], rank, world)
    return Y[lo:hi]


class Collectives:
    """The collectives of the sharded schedule, on the current stream.

    At world size 1 they are local copies; FCB_FORCE_COLLECTIVES=1 issues the
    NCCL calls anyway (a one-rank group), so the stream ordering between the
    collectives and the device steps is exercised on a single GPU.
    """

    def __init__(self, group=None):
        self.group = group
        self.rank, self.world = _world(group)
        self.force = (os.environ.get("FCB_FORCE_COLLECTIVES", "0") != "0"
                      and group is not None and dist.is_initialized())

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        """out (world * inp.numel()) <- concatenation of every rank's inp."""
        if self.world == 1 and not self.force:
            out.view(-1)[: inp.numel()].copy_(inp.view(-1))
            return
        dist.all_gather_into_tensor(out.view(-1), inp.contiguous().view(-1), group=self.group)

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1 or self.force:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t


# ---------------------------------------------------------------------------
# device steps (C ABI)
# ---------------------------------------------------------------------------
class DeviceOps:
    """The C-ABI steps of csrc/shard.cu, on the current torch stream."""

    def __init__(self):
        self.lib = _lib.load()
        self.dev = _dev.require_cuda()

    def _call(self, name, *args):
        _lib.check(getattr(self.lib, name)(*args), name)

    # buffers -------------------------------------------------------------
    def zeros(self, shape, dtype=torch.float64):
        return torch.zeros(shape, dtype=dtype, device=self.dev)

    def tensor(self, a):
        return _dev.f64(a, self.dev)

    def snapshot(self, src: torch.Tensor, dst: torch.Tensor):
        """Asynchronous copy of a control word to pinned host memory + event."""
        dst.copy_(src, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return ev

    def pinned_int(self):
        return torch.zeros(1, dtype=torch.int32, pin_memory=True)

    # steps -----------------------------------------------------------------
    def point_sums(self, P: torch.Tensor, out: torch.Tensor) -> None:
        n, d = P.shape
        self._call("fcb_point_sums", _dev.ptr(P), n, d, _dev.ptr(out), _dev.stream())

    def workspace(self, nbytes: int, tag: str) -> torch.Tensor:
        return _dev.Workspace.get(nbytes, tag)

    def lse_sweep(self, prec, R, S, scal, pot, scale, shift, out, bary, gate, tag,
                  est=None, est_logw=0.0):
        nr, d = R.shape
        ns = S.shape[0]
        ws = self.workspace(self.lib.fcb_lse_sweep_workspace_bytes(prec, nr, ns, d), tag)
        self._call("fcb_lse_sweep", prec, _dev.ptr(R), nr, _dev.ptr(S), ns, d, _dev.ptr(scal),
                   _dev.ptr(pot), _dev.ptr(est), float(est_logw), float(scale), float(shift),
                   _dev.ptr(out), _dev.ptr(bary), _dev.ptr(gate), _dev.ptr(ws), ws.numel(),
                   _dev.stream())

    def shard_init(self, prec, X, ysum, omega_fixed, warm_f, warm_p, warm_valid, scal_x, scal_s,
                   f, p, ctl, eslot, plan_state):
        n, d = X.shape
        self._call("fcb_shard_init", prec, _dev.ptr(X), n, d, _dev.ptr(ysum), float(omega_fixed),
                   _dev.ptr(warm_f), _dev.ptr(warm_p), _dev.ptr(warm_valid), _dev.ptr(scal_x),
                   _dev.ptr(scal_s), _dev.ptr(f), _dev.ptr(p), _dev.ptr(ctl), _dev.ptr(eslot),
                   _dev.ptr(plan_state), _dev.stream())

    def cross_merge(self, n, d, R, gath, scal, tol, max_iters, f, fnext, rs, mass, ybar, ctl,
                    eslot, stat):
        self._call("fcb_shard_cross_merge", n, d, R, _dev.ptr(gath), _dev.ptr(scal), float(tol),
                   int(max_iters), _dev.ptr(f), _dev.ptr(fnext), _dev.ptr(rs), _dev.ptr(mass),
                   _dev.ptr(ybar), _dev.ptr(ctl), _dev.ptr(eslot), _dev.ptr(stat), _dev.stream())

    def self_rows(self, n, d, row0, nown, Lb, scal, p, send, ctl):
        self._call("fcb_shard_self_rows", n, d, row0, nown, _dev.ptr(Lb), _dev.ptr(scal),
                   _dev.ptr(p), _dev.ptr(send), _dev.ptr(ctl), _dev.stream())

    def self_commit(self, n, d, R, chunk, gath, tol, max_iters, p, pnext, rho, massp, xbar, ctl,
                    eslot, stat):
        self._call("fcb_shard_self_commit", n, d, R, chunk, _dev.ptr(gath), float(tol),
                   int(max_iters), _dev.ptr(p), _dev.ptr(pnext), _dev.ptr(rho), _dev.ptr(massp),
                   _dev.ptr(xbar), _dev.ptr(ctl), _dev.ptr(eslot), _dev.ptr(stat), _dev.stream())

    def flow_finish(self, X, rs, mass, ybar, rho, massp, xbar, stat_x, stat_p, tol, f, p, warm_f,
                    warm_p, warm_valid, flow, fstat, scal, plan_state, iteration, flow_log,
                    conv_tol, ctl):
        n, d = X.shape
        ws = self.workspace(self.lib.fcb_shard_finish_workspace_bytes(n), "shard_fin")
        self._call("fcb_shard_flow_finish", _dev.ptr(X), n, d, _dev.ptr(rs), _dev.ptr(mass),
                   _dev.ptr(ybar), _dev.ptr(rho), _dev.ptr(massp), _dev.ptr(xbar),
                   _dev.ptr(stat_x), _dev.ptr(stat_p), float(tol), _dev.ptr(f), _dev.ptr(p),
                   _dev.ptr(warm_f), _dev.ptr(warm_p), _dev.ptr(warm_valid), _dev.ptr(flow),
                   _dev.ptr(fstat), _dev.ptr(scal), _dev.ptr(plan_state), int(iteration),
                   _dev.ptr(flow_log), float(conv_tol), _dev.ptr(ctl), _dev.ptr(ws), ws.numel(),
                   _dev.stream())

    # SVGD ------------------------------------------------------------------
    def mixture_params(self, q):
        return q.num_components, q.device_params()

    def median_bandwidth(self, X, hstat, gate):
        n, d = X.shape
        ws = self.workspace(self.lib.fcb_median_workspace_bytes(n), "shard_med")
        self._call("fcb_median_bandwidth", _dev.ptr(X), n, d, math.log(n + 1.0), _dev.ptr(hstat),
                   _dev.ptr(gate), _dev.ptr(ws), ws.numel(), _dev.stream())

    def median_sharded(self, X, hstat, gate, coll):
        """median_bandwidth (stein.py:66-76) over this rank's pair tiles, the radix
        histograms all-reduced per pass (fcb_median_shard_*)."""
        n, d = X.shape
        if n < 2:
            return self.median_bandwidth(X, hstat, gate)
        ws = self.workspace(self.lib.fcb_median_workspace_bytes(n), "shard_med")
        lo, hi = shard_bounds(int(self.lib.fcb_median_tiles(n)), coll.rank, coll.world)
        off = int(self.lib.fcb_median_hist_offset())
        hist = ws[off:off + 2 * 2048 * 8].view(torch.int64)
        s = _dev.stream()
        self._call("fcb_median_shard_init", n, _dev.ptr(ws), ws.numel(), _dev.ptr(gate), s)
        for p in range(6):
            self._call("fcb_median_shard_pass", _dev.ptr(X), n, d, p, lo, hi, _dev.ptr(ws),
                       _dev.ptr(gate), s)
            coll.all_reduce_sum(hist)
            self._call("fcb_median_shard_select", n, p, _dev.ptr(ws), _dev.ptr(gate), s)
        self._call("fcb_median_shard_finish", n, math.log(n + 1.0), _dev.ptr(hstat),
                   _dev.ptr(ws), _dev.ptr(gate), s)

    def gmm_score(self, X, k, params, out, gate):
        n, d = X.shape
        self._call("fcb_gmm_eval", _dev.ptr(X), n, d, k, _dev.ptr(params), _dev.ptr(out), None,
                   _dev.ptr(gate), _dev.stream())

    def stein_partial(self, prec, X, col0, ncols, scores, hstat, part, gate):
        n, d = X.shape
        ws = self.workspace(self.lib.fcb_stein_partial_workspace_bytes(prec, n, ncols, d),
                            "shard_sv")
        self._call("fcb_stein_partial", prec, _dev.ptr(X), n, d, col0, ncols, _dev.ptr(scores),
                   _dev.ptr(hstat), _dev.ptr(part), _dev.ptr(gate), _dev.ptr(ws), ws.numel(),
                   _dev.stream())

    def stein_combine(self, X, R, parts, hstat, flow, fstat, plan_state, iteration, flow_log,
                      conv_tol):
        n, d = X.shape
        ws = self.workspace(self.lib.fcb_stein_combine_workspace_bytes(n), "shard_svc")
        self._call("fcb_stein_combine", _dev.ptr(X), n, d, R, _dev.ptr(parts), _dev.ptr(hstat),
                   _dev.ptr(flow), _dev.ptr(fstat), _dev.ptr(plan_state), int(iteration),
                   _dev.ptr(flow_log), float(conv_tol), _dev.ptr(ws), ws.numel(), _dev.stream())


# ---------------------------------------------------------------------------
# the sharded Sinkhorn flow
# ---------------------------------------------------------------------------
class _Poller:
    """Lagged completion polls of a device control word: the host queues up to
    `lag` iterations past the last one it has seen complete."""

    def __init__(self, ops, word: torch.Tensor, lag: int = 2):
        self.ops, self.word, self.lag = ops, word, lag
        self.pending: collections.deque = collections.deque()
        self.pool = [ops.pinned_int() for _ in range(lag + 2)]
        self.k = 0

    def after_iteration(self) -> bool:
        """Snapshot the word; True once a completed snapshot shows it set."""
        snap = self.pool[self.k % len(self.pool)]
        self.k += 1
        self.pending.append((self.ops.snapshot(self.word, snap), snap))
        while len(self.pending) > self.lag:
            ev, s = self.pending.popleft()
            ev.synchronize()
            if int(s[0]) != 0:
                return True
        return False


class ShardedSinkhorn:
    """sinkhorn_flow (sinkhorn.py:338-400) over reference samples sharded across
    the ranks of `group`, device-resident (see the module docstring).

    Y_local: this rank's shard (device tensor or host array, float64 (m_r, d)).
    n: number of flow points (trajectory states) the instance is sized for.
    """

    def __init__(self, Y_local, n: int, cfg: SinkhornConfig = SinkhornConfig(), group=None,
                 ops=None, precision: Optional[int] = None, lag: int = 2):
        self.ops = ops or DeviceOps()
        self.coll = Collectives(group)
        self.cfg = cfg
        ops = self.ops
        self.Y = Y_local if isinstance(Y_local, torch.Tensor) else ops.tensor(Y_local)
        self.Y = self.Y.contiguous()
        m_r, d = self.Y.shape
        self.n, self.d = n, d
        R, rank = self.coll.world, self.coll.rank
        # global Y statistics (d sums, sum of squares, count): one all_reduce
        self.ysum = ops.zeros((d + 2,))
        ops.point_sums(self.Y, self.ysum)
        self.coll.all_reduce_sum(self.ysum)
        m_all = torch.tensor([float(m_r)], dtype=torch.float64)
        if R > 1:
            m_all = m_all.to(self.ysum.device)
            self.coll.all_reduce_sum(m_all)
        self.m_global = int(round(float(m_all.item())))
        # precision from the GLOBAL shape, identical on every rank
        self.prec = (precision if precision is not None else
                     _precision.pick(cfg.precision, n * max(n, self.m_global), cfg.tol))
        self.logb = -math.log(self.m_global)
        self.loga = -math.log(n)
        self.log_frac = math.log(max(m_r, 1) / self.m_global)
        self.rows = shard_bounds(n, rank, R)
        self.nown = self.rows[1] - self.rows[0]
        self.chunk = (n + R - 1) // R
        z = ops.zeros
        self.f, self.fnext, self.p, self.pnext = z((n,)), z((n,)), z((n,)), z((n,))
        self.g = z((m_r,))
        self.send_x = z((n, d + 1))
        self.gath_x = z((R, n, d + 1))
        self.rs, self.mass, self.ybar = z((n,)), z((n,)), z((n, d))
        self.rho, self.massp, self.xbar = z((n,)), z((n,)), z((n, d))
        self.Lb = z((max(self.nown, 1), d + 1))
        self.send_s = z((self.chunk, d + 4))
        self.gath_s = z((R, self.chunk, d + 4))
        self.scal_x, self.scal_s = z((16,)), z((16,))
        self.stat_x, self.stat_p = z((4,)), z((4,))
        self.ctl = z((8,), dtype=torch.int32)
        self.eslot = z((2,), dtype=torch.int64)
        self.lag = lag
        self.iters_queued = (0, 0)

    # one inner iteration of each solve ------------------------------------
    def _cross_iteration(self, X):
        ops, cfg, d = self.ops, self.cfg, self.d
        gate = self.ctl[0:1]
        # g_r = w (log b - LSE_rows(Y_r vs X; f)); rows shifted by the last g
        ops.lse_sweep(self.prec, self.Y, X, self.scal_x, self.f, 1.0, self.logb, self.g, None,
                      gate, "shard_sw", est=self.g, est_logw=self.logb)
        # {L_r, ybar_r} of rows X vs Y_r under g_r, gathered over ranks; the
        # shard's LSE is ~ log(m_r / M) below the full one, log a - f / w
        ops.lse_sweep(self.prec, X, self.Y, self.scal_x, self.g, 0.0, 0.0, None, self.send_x,
                      gate, "shard_sw", est=self.f, est_logw=self.loga + self.log_frac)
        self.coll.all_gather(self.gath_x, self.send_x)
        ops.cross_merge(self.n, d, self.coll.world, self.gath_x, self.scal_x, cfg.tol,
                        cfg.max_iters, self.f, self.fnext, self.rs, self.mass, self.ybar,
                        self.ctl, self.eslot, self.stat_x)

    def _self_iteration(self, X):
        ops, cfg, d = self.ops, self.cfg, self.d
        gate = self.ctl[1:2]
        lo, hi = self.rows
        if self.nown > 0:
            ops.lse_sweep(self.prec, X[lo:hi], X, self.scal_s, self.p, 0.0, 0.0, None, self.Lb,
                          gate, "shard_sw", est=self.p[lo:hi], est_logw=self.loga)
            ops.self_rows(self.n, d, lo, self.nown, self.Lb, self.scal_s, self.p, self.send_s,
                          self.ctl)
        self.coll.all_gather(self.gath_s, self.send_s)
        ops.self_commit(self.n, d, self.coll.world, self.chunk, self.gath_s, cfg.tol,
                        cfg.max_iters, self.p, self.pnext, self.rho, self.massp, self.xbar,
                        self.ctl, self.eslot, self.stat_p)

    def _solve(self, step, word: torch.Tensor) -> int:
        poll = _Poller(self.ops, word, self.lag)
        queued = 0
        for _ in range(self.cfg.max_iters):
            step()
            queued += 1
            if queued < self.cfg.max_iters and poll.after_iteration():
                break
        return queued

    def flow_into(self, X: torch.Tensor, warm_f, warm_p, warm_valid, flow, fstat,
                  plan_state=None, iteration: int = 0, flow_log=None, conv_tol: float = 0.0):
        """Device-resident flow on X (n, d): writes flow and fstat (layout of
        fcb_sinkhorn_flow) and the planner hooks; never synchronises with the
        host except through the lagged loop polls."""
        ops, cfg = self.ops, self.cfg
        ops.shard_init(self.prec, X, self.ysum, _omega_arg(cfg.omega), warm_f, warm_p, warm_valid,
                       self.scal_x, self.scal_s, self.f, self.p, self.ctl, self.eslot, plan_state)
        qx = self._solve(lambda: self._cross_iteration(X), self.ctl[0:1])
        qp = self._solve(lambda: self._self_iteration(X), self.ctl[1:2])
        self.iters_queued = (qx, qp)
        ops.flow_finish(X, self.rs, self.mass, self.ybar, self.rho, self.massp, self.xbar,
                        self.stat_x, self.stat_p, cfg.tol, self.f, self.p, warm_f, warm_p,
                        warm_valid, flow, fstat, self.scal_x, plan_state, iteration, flow_log,
                        conv_tol, self.ctl)


class ShardedSinkhornFlow:
    """Host-facing sinkhorn_flow over sharded reference samples, keeping the
    warm potentials (f, p) between calls like SinkhornWarmState."""

    def __init__(self, Y_local, cfg: SinkhornConfig = SinkhornConfig(), group=None, ops=None):
        self.ops = ops or DeviceOps()
        self.Y_local = np.asarray(Y_local, dtype=np.float64)
        self.cfg, self.group = cfg, group
        self.solver: Optional[ShardedSinkhorn] = None
        self.warm = None

    def __call__(self, X, stats: dict | None = None) -> FlowField:
        X = np.atleast_2d(np.asarray(X, dtype=np.float64))
        n, d = X.shape
        ops = self.ops
        if self.solver is None or self.solver.n != n:
            self.solver = ShardedSinkhorn(self.Y_local, n, self.cfg, self.group, ops)
            self.warm = (ops.zeros((n,)), ops.zeros((n,)), ops.zeros((2,), dtype=torch.int32))
        Xd = ops.tensor(X)
        flow, fstat = ops.zeros((n, d)), ops.zeros((8,))
        wf, wp, wv = self.warm
        self.solver.flow_into(Xd, wf, wp, wv, flow, fstat)
        st = fstat.cpu().numpy()
        if stats is not None:
            stats.update(omega=float(st[4]), iters_cross=int(st[5]), iters_self=int(st[6]),
                         worst=float(st[0]))
        if st[2] != 0.0:
            raise FlowError(flow_error_message(float(st[0]), self.cfg.tol))
        return FlowField(a=flow.cpu().numpy(), converged=bool(st[1] != 0.0),
                         marginal_error=float(st[0]))


# ---------------------------------------------------------------------------
# source-sharded SVGD
# ---------------------------------------------------------------------------
class ShardedStein:
    """stein_flow (stein.py:79-122) with the sources split across ranks.

    The bandwidth is fixed (SteinConfig.bandwidth > 0) or the exact median,
    whose pair tiles are split across the ranks with the radix histograms
    all-reduced per pass (identical on every rank).
    """

    def __init__(self, n: int, d: int, q, bandwidth, group=None, ops=None,
                 precision: Optional[int] = None, stein_precision: str = "auto"):
        self.ops = ops or DeviceOps()
        self.coll = Collectives(group)
        R, rank = self.coll.world, self.coll.rank
        self.n, self.d = n, d
        self.cols = shard_bounds(n, rank, R)
        self.k, self.params = self.ops.mixture_params(q)
        self.bandwidth = bandwidth
        self.prec = precision if precision is not None else _precision.pick(stein_precision, n * n)
        z = self.ops.zeros
        self.hstat = z((4,))
        if bandwidth != "median":
            h = float(bandwidth)
            self.hstat.copy_(torch.tensor([max(h, 1e-12), float("nan"), float(h <= 1e-12), 0.0],
                                          dtype=torch.float64))
        self.scores = z((n, d))
        self.part = z((n, d + 1))
        self.parts = z((R, n, d + 1))

    def flow_into(self, X, flow, fstat=None, plan_state=None, iteration: int = 0, flow_log=None,
                  conv_tol: float = 0.0):
        ops = self.ops
        if self.bandwidth == "median":
            ops.median_sharded(X, self.hstat, plan_state, self.coll)
        ops.gmm_score(X, self.k, self.params, self.scores, plan_state)
        lo, hi = self.cols
        if hi > lo:
            ops.stein_partial(self.prec, X, lo, hi - lo, self.scores, self.hstat, self.part,
                              plan_state)
        self.coll.all_gather(self.parts, self.part)
        ops.stein_combine(X, self.coll.world, self.parts, self.hstat, flow, fstat, plan_state,
                          iteration, flow_log, conv_tol)


# ---------------------------------------------------------------------------
# batched independent problems (BASELINE config 5)
# ---------------------------------------------------------------------------
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
