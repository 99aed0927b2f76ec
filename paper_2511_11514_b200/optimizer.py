"""The coverage-planning loop, run on device (drop-in for reference optimizer.py).

Each iteration rolls the controls out, evaluates the statistical flow on the
workspace points, projects it through the flow-matching LQR and steps
U <- clamp(U + eta v*) -- the reference's loop body (optimizer.py:221-269).
Here the body is a fixed sequence of stream-ordered device calls with no
host synchronisation: convergence, FlowError and rollout/Riccati blow-ups are
recorded in a device status word that gates every later kernel, and the host
only polls completed events to stop queueing work.  Inputs cross to the
device once (targets, initial controls) and the PlanResult crosses back once.
"""

from __future__ import annotations

import collections
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import numpy.typing as npt
import torch

from . import _dev, _lib, _precision
from .dynamics import (
    Discretization,
    DynamicsModel,
    RolloutDivergenceError,
    Trajectory,
    device_model,
    rollout,
    rollout_method,
)
from .lqr import RiccatiDivergenceError, workspace_weights
from .reference import GaussianMixture, ReferenceDistribution, SamplePoints, to_sample_based
from .seeding import STREAM_INIT_CONTROLS, STREAM_METRIC, STREAM_REFERENCE, rng_stream
from .sinkhorn import (
    FlowError,
    SinkhornConfig,
    _check_cost_finite,
    _omega_arg,
    flow_error_message,
    sinkhorn_divergence,
)
from .stein import SteinConfig

METHODS = ("stein", "sinkhorn")


@dataclass(frozen=True)
class PlanConfig:
    method: str = "stein"
    eta: float = 0.1
    max_iterations: int = 300
    convergence_tol: float = 1e-4
    control_clamp: tuple[float, ...] | None = None
    seed: int = 0
    initial_controls: str | np.ndarray = "random_small"
    init_scale: float = 1e-2
    metric_interval: int = 10
    metric_samples: int | None = None
    q_weight: float = 1.0
    r_weight: float = 0.1
    stein: SteinConfig = field(default_factory=SteinConfig)
    sinkhorn: SinkhornConfig = field(default_factory=SinkhornConfig)
    workers: int | None = None

    def __post_init__(self) -> None:
        if self.method not in METHODS:
            raise ValueError(f"method must be one of {METHODS}, got {self.method!r}")
        if not self.eta > 0:
            raise ValueError(f"eta must be positive, got {self.eta}")
        if self.max_iterations < 1:
            raise ValueError(f"max_iterations must be >= 1, got {self.max_iterations}")
        if self.convergence_tol < 0:
            raise ValueError(f"convergence_tol must be >= 0, got {self.convergence_tol}")
        if isinstance(self.initial_controls, str):
            if self.initial_controls not in ("random_small", "zeros"):
                raise ValueError(
                    'initial_controls must be "random_small", "zeros", or a control array, '
                    f"got {self.initial_controls!r}"
                )
        if not self.init_scale > 0:
            raise ValueError(f"init_scale must be positive, got {self.init_scale}")
        if self.metric_interval < 0:
            raise ValueError(f"metric_interval must be >= 0, got {self.metric_interval}")
        if self.metric_samples is not None and self.metric_samples < 1:
            raise ValueError(f"metric_samples must be >= 1, got {self.metric_samples}")
        if self.control_clamp is not None:
            clamp = tuple(float(c) for c in self.control_clamp)
            if any(c <= 0 for c in clamp):
                raise ValueError("control_clamp bounds must be positive")
            object.__setattr__(self, "control_clamp", clamp)


@dataclass(frozen=True)
class PhaseTimes:
    """Seconds per phase (device time from CUDA events; total is wall clock)."""

    flow: float
    lqr: float
    rollout: float
    total: float


@dataclass(frozen=True)
class PlanResult:
    trajectory: Trajectory
    converged: bool
    iterations_used: int
    flow_norms: npt.NDArray[np.float64]
    lqr_costs: npt.NDArray[np.float64]
    metric_iterations: tuple[int, ...]
    metric_values: tuple[float, ...]
    phase_times: PhaseTimes
    final_metric: float | None


class PlanError(RuntimeError):
    """A planning phase failed; carries the iteration and last good trajectory."""

    def __init__(self, stage: str, iteration: int, trajectory: Trajectory | None, cause: Exception):
        self.stage = stage
        self.iteration = iteration
        self.trajectory = trajectory
        super().__init__(f"{stage} failed at iteration {iteration}: {cause}")


def coverage_metric(
    S, model: DynamicsModel, q_samples, cfg: SinkhornConfig = SinkhornConfig(),
    workers: int | None = None,
) -> float:
    """Divergence between project(S[1:]) and target draws (optimizer.py:126-139)."""
    S = np.asarray(S, dtype=np.float64)
    return sinkhorn_divergence(model.project_states(S[1:]), q_samples, cfg, workers=workers)


def initial_controls(cfg: PlanConfig, model: DynamicsModel, num_steps: int) -> np.ndarray:
    """U0: provided array, zeros, or init_scale * N(0,1) from stream [seed, 1]."""
    shape = (num_steps, model.control_dim)
    if isinstance(cfg.initial_controls, np.ndarray):
        U0 = np.asarray(cfg.initial_controls, dtype=np.float64)
        if U0.shape != shape:
            raise ValueError(f"provided controls must have shape {shape}, got {U0.shape}")
        return U0.copy()
    if cfg.initial_controls == "zeros":
        return np.zeros(shape)
    return cfg.init_scale * rng_stream(cfg.seed, STREAM_INIT_CONTROLS).standard_normal(shape)


def metric_targets(q: ReferenceDistribution, cfg: PlanConfig, num_steps: int) -> np.ndarray:
    m = cfg.metric_samples if cfg.metric_samples is not None else num_steps
    return q.sample(m, [cfg.seed, STREAM_METRIC])


# ---------------------------------------------------------------------------
# the device loop
# ---------------------------------------------------------------------------
class _Events:
    """Per-iteration CUDA events for phase timing."""

    def __init__(self) -> None:
        self.rows: list[tuple] = []

    def mark(self) -> torch.cuda.Event:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev


@dataclass
class PlanRun:
    """Device-side record of one plan() call (used by bench.py and tests)."""

    result: PlanResult | None = None
    flow_log: np.ndarray | None = None  # (iterations_used, 4)
    precision: int = 0
    pairs: float = 0.0  # executed (query, source) pair evaluations in the flows
    launches: int = 0


def _pair_count(method: str, log: np.ndarray, T: int, M: int) -> float:
    if method != "sinkhorn" or log.size == 0:
        return float(log.shape[0]) * T * T if method == "stein" else 0.0
    ka, ks = log[:, 1], log[:, 2]
    return float((2.0 * ka * T * M + ks * T * T).sum())


def plan(
    model: DynamicsModel,
    q: ReferenceDistribution,
    disc: Discretization,
    cfg: PlanConfig = PlanConfig(),
    *,
    group=None,
) -> PlanResult:
    """Synthesize a coverage trajectory for q (optimizer.py:171-304).

    group (additive, keyword-only): shard the flow over the ranks of a
    torch.distributed group (one GPU each); see plan_detailed.
    """
    return plan_detailed(model, q, disc, cfg, group=group).result


def plan_detailed(
    model: DynamicsModel,
    q: ReferenceDistribution,
    disc: Discretization,
    cfg: PlanConfig = PlanConfig(),
    poll_lag: int = 2,
    resident_targets: torch.Tensor | None = None,
    group=None,
) -> PlanRun:
    """plan() plus the device-side record (inner iteration log, pair count).

    resident_targets: the transport targets already in device memory
    (float64, (M, d)); used by bench.py to time with inputs resident in HBM.
    With `group`, this rank's shard of them.
    group (additive, keyword): a torch.distributed process group, one rank per
    GPU.  Every rank passes the same problem; the Sinkhorn reference samples
    (or the SVGD sources) are sharded across the ranks (distributed.py) and
    every rank returns the same PlanResult.  Rollout and LQR are replicated.
    """
    if cfg.method == "stein" and not isinstance(q, GaussianMixture):
        raise ValueError("the stein method needs a score-based (mixture) reference")
    if disc.s0.shape != (model.state_dim,):
        raise ValueError(f"s0 must have shape ({model.state_dim},), got {disc.s0.shape}")

    T = disc.num_steps
    if cfg.method == "sinkhorn":
        targets = q if isinstance(q, SamplePoints) else to_sample_based(
            q, T, [cfg.seed, STREAM_REFERENCE]
        )
    else:
        targets = None
    weights = workspace_weights(model.project_matrix, model.control_dim, cfg.q_weight, cfg.r_weight)
    want_metric = cfg.metric_interval > 0
    # metric draws from a point cloud are a device gather of host-drawn indices
    # from the targets already on the device (below); mixtures draw on the host
    metric_gather = (want_metric and isinstance(q, SamplePoints) and cfg.method == "sinkhorn"
                     and group is None)
    q_metric = metric_targets(q, cfg, T) if want_metric and not metric_gather else None

    U0 = initial_controls(cfg, model, T)
    clamp = cfg.control_clamp
    if clamp is not None and len(clamp) != model.control_dim:
        raise ValueError(f"control_clamp needs {model.control_dim} bounds, got {len(clamp)}")
    bounds = np.asarray(clamp, dtype=np.float64) if clamp is not None else None
    if bounds is not None:
        np.clip(U0, -bounds, bounds, out=U0)

    spec = device_model(model)
    linear_model = spec.model_id in (
        _lib.FCB_MODEL_SINGLE_INTEGRATOR_2D, _lib.FCB_MODEL_DOUBLE_INTEGRATOR_2D, _lib.FCB_MODEL_LTI
    )
    d = model.workspace_dim
    if d > 3:
        raise NotImplementedError("device flows support workspaces of dimension 1-3")
    n_s, m_c = model.state_dim, model.control_dim
    maxit = cfg.max_iterations
    lib = _lib.load()
    dev = _dev.require_cuda()
    stream = _dev.stream()
    t_begin = time.perf_counter()

    # ---- one-time uploads ------------------------------------------------
    s0 = _dev.f64(disc.s0, dev)
    Ubuf = [_dev.f64(U0, dev), _dev.zeros((T, m_c), device=dev)]
    Sbuf = [_dev.zeros((T + 1, n_s), device=dev), _dev.zeros((T + 1, n_s), device=dev)]
    X = _dev.zeros((T, d), device=dev)
    flow = _dev.zeros((T, d), device=dev)
    P = _dev.f64(model.project_matrix, dev)
    Q = _dev.f64(weights.Q, dev)
    R = _dev.f64(weights.R, dev)
    clamp_d = _dev.f64(bounds, dev) if bounds is not None else None
    prm = spec.device_params(dev)
    state = torch.zeros(8, dtype=torch.int32, device=dev)
    flow_log = _dev.zeros((maxit, 4), device=dev)
    lqr_costs = _dev.zeros((maxit,), device=dev)
    fstat = _dev.zeros((8,), device=dev)
    n_metric = (maxit + cfg.metric_interval - 1) // cfg.metric_interval if want_metric else 0
    metric_vals = _dev.zeros((max(n_metric, 1), 4), device=dev)
    status_host = torch.zeros(8, dtype=torch.int32, pin_memory=True)

    sharded = group is not None
    if sharded:
        from . import distributed as _dist

        g_rank, g_world = _dist._world(group)
    if cfg.method == "sinkhorn":
        Y = targets.points
        if Y.shape[1] != d:
            from .sinkhorn import SinkhornInputError

            raise SinkhornInputError(f"point dims disagree: {d} vs {Y.shape[1]}")
        M = Y.shape[0]
        scfg = cfg.sinkhorn
        prec = _precision.pick(scfg.precision, T * max(T, M), scfg.tol)
        warm_f, warm_p = _dev.zeros((T,), device=dev), _dev.zeros((T,), device=dev)
        warm_valid = torch.zeros(2, dtype=torch.int32, device=dev)
        omega_fixed = _omega_arg(scfg.omega)
        if sharded:
            Yd = (resident_targets if resident_targets is not None
                  else _dev.f64(_dist.shard_rows(Y, g_rank, g_world), dev))
            shard_flow = _dist.ShardedSinkhorn(Yd, T, scfg, group, precision=prec)
        else:
            Yd = resident_targets if resident_targets is not None else _dev.f64(Y, dev)
            flow_ws = _dev.Workspace.get(lib.fcb_sinkhorn_flow_workspace_bytes(prec, T, M, d),
                                         "plan_flow")
    else:
        M = 0
        scfg_st = cfg.stein
        prec = _precision.pick(scfg_st.precision, T * T)
        gmm = q.device_params()
        bw_fixed = 0.0 if scfg_st.bandwidth == "median" else float(scfg_st.bandwidth)
        log_np1 = math.log(T + 1.0)
        if sharded:
            shard_flow = _dist.ShardedStein(T, d, q, scfg_st.bandwidth, group, precision=prec)
        else:
            flow_ws = _dev.Workspace.get(lib.fcb_stein_flow_full_workspace_bytes(prec, T, d),
                                         "plan_flow")
    upd_ws = _dev.Workspace.get(lib.fcb_plan_update_workspace_bytes(n_s, m_c, T), "plan_upd")
    roll_ws = _dev.Workspace.get(lib.fcb_rollout_workspace_bytes(n_s, T), "plan_roll")
    if want_metric:
        if metric_gather:
            Mm = cfg.metric_samples if cfg.metric_samples is not None else T
            Ymd = q.sample_device(Mm, [cfg.seed, STREAM_METRIC], points=Yd)
        else:
            Ym = np.atleast_2d(np.asarray(q_metric, dtype=np.float64))
            Mm = Ym.shape[0]
            Ymd = _dev.f64(Ym, dev)
        mprec = _precision.pick(cfg.sinkhorn.precision, max(T, Mm) ** 2, cfg.sinkhorn.tol)
        met_ws = _dev.Workspace.get(
            lib.fcb_sinkhorn_divergence_workspace_bytes(mprec, T, Mm, d), "plan_metric"
        )
        # OT(Y, Y) of the metric draws: solved once per omega (a numeric
        # SinkhornConfig.omega makes every later metric skip the M x M solve)
        yy_cache = torch.zeros(5, dtype=torch.float64, device=dev)

    launches0 = lib.fcb_launch_count()
    marks: list[tuple] = []
    pending: collections.deque = collections.deque()
    state_ptr = _dev.ptr(state)

    def call(name, *args):
        rc = getattr(lib, name)(*args)
        _lib.check(rc, name)

    ring = [torch.zeros(8, dtype=torch.int32, pin_memory=True) for _ in range(poll_lag + 2)]
    # status snapshots every `poll_every` iterations: after a stop, the queued
    # kernels are gated by the device status word and exit at once
    poll_every = 8
    e_prev = None
    # linear models with the on-chip flow: iterations 1.. run as one
    # persistent launch (fcb_plan_fused) after iteration 0 has stored the
    # Riccati phase; anything it does not cover stays on the per-iteration path
    fused_ok = (os.environ.get("FCB_FUSED", "1") != "0" and cfg.method == "sinkhorn"
                and not want_metric and prec == _lib.FCB_FP32 and not sharded
                and d == 2 and maxit > 1 and spec.model_id in (
                    _lib.FCB_MODEL_SINGLE_INTEGRATOR_2D, _lib.FCB_MODEL_DOUBLE_INTEGRATOR_2D))
    # the same for the SVGD flow (fcb_plan_fused_stein, fp64 sweeps): iterations
    # 1.. in one cooperative launch
    fused_stein_ok = (os.environ.get("FCB_FUSED", "1") != "0" and cfg.method == "stein"
                      and not want_metric and prec == _lib.FCB_FP64 and not sharded
                      and d == 2 and maxit > 1 and spec.model_id in (
                          _lib.FCB_MODEL_SINGLE_INTEGRATOR_2D,
                          _lib.FCB_MODEL_DOUBLE_INTEGRATOR_2D))
    fused_ran = False
    phase_ns = (torch.zeros(3, dtype=torch.int64, device=dev)
                if (fused_ok or fused_stein_ok) else None)
    for it in range(maxit):
        cur = it & 1
        if it == 1 and fused_ok:
            _dev.nvtx_push("fused_loop")
            fws = _dev.Workspace.get(
                lib.fcb_plan_fused_workspace_bytes(1, T, M, d, m_c), "plan_fused")
            rc = lib.fcb_plan_fused(
                spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(s0), _dev.ptr(Ubuf[0]),
                _dev.ptr(Ubuf[1]), _dev.ptr(Sbuf[0]), _dev.ptr(Sbuf[1]), T, float(disc.dt), d,
                _dev.ptr(P), _dev.ptr(X), _dev.ptr(flow), _dev.ptr(Q), _dev.ptr(R),
                float(cfg.eta), _dev.ptr(clamp_d), _dev.ptr(Yd), M, omega_fixed, scfg.max_iters,
                scfg.tol, float(cfg.convergence_tol), _dev.ptr(warm_f), _dev.ptr(warm_p),
                _dev.ptr(warm_valid), _dev.ptr(fstat), state_ptr, _dev.ptr(flow_log),
                _dev.ptr(lqr_costs), _dev.ptr(phase_ns), 1, maxit, 1, _dev.ptr(upd_ws),
                _dev.ptr(fws), fws.numel(), stream)
            _dev.nvtx_pop()
            if rc == _lib.FCB_OK:
                fused_ran = True
                break
            if rc != _lib.FCB_ENOTSUP:
                _lib.check(rc, "fcb_plan_fused")
        if it == 1 and fused_stein_ok:
            _dev.nvtx_push("fused_loop")
            sws = _dev.Workspace.get(lib.fcb_plan_fused_stein_workspace_bytes(T, d, m_c),
                                     "plan_fused_stein")
            rc = lib.fcb_plan_fused_stein(
                spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(s0), _dev.ptr(Ubuf[0]),
                _dev.ptr(Ubuf[1]), _dev.ptr(Sbuf[0]), _dev.ptr(Sbuf[1]), T, float(disc.dt), d,
                _dev.ptr(P), _dev.ptr(X), _dev.ptr(flow), _dev.ptr(Q), _dev.ptr(R),
                float(cfg.eta), _dev.ptr(clamp_d), q.num_components, _dev.ptr(gmm), bw_fixed,
                log_np1, float(cfg.convergence_tol), _dev.ptr(fstat), state_ptr,
                _dev.ptr(flow_log), _dev.ptr(lqr_costs), _dev.ptr(phase_ns), 1, maxit,
                _dev.ptr(upd_ws), _dev.ptr(sws), sws.numel(), stream)
            _dev.nvtx_pop()
            if rc == _lib.FCB_OK:
                fused_ran = True
                break
            if rc != _lib.FCB_ENOTSUP:
                _lib.check(rc, "fcb_plan_fused_stein")
        if e_prev is None:
            e_prev = torch.cuda.Event(enable_timing=True)
            e_prev.record()
        e0 = e_prev  # the previous iteration's end event
        _dev.nvtx_push("rollout")
        call("fcb_rollout", spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(s0),
             _dev.ptr(Ubuf[cur]), T, float(disc.dt), _dev.ptr(Sbuf[cur]), d, _dev.ptr(P),
             _dev.ptr(X), None, state_ptr, it, 1, _dev.ptr(roll_ws), stream)
        _dev.nvtx_pop()
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        e2 = e1
        if want_metric and it % cfg.metric_interval == 0:
            call("fcb_sinkhorn_divergence_cached", mprec, _dev.ptr(X), T, _dev.ptr(Ymd), Mm, d,
                 _omega_arg(cfg.sinkhorn.omega), cfg.sinkhorn.max_iters, cfg.sinkhorn.tol,
                 _dev.ptr(metric_vals[it // cfg.metric_interval]), state_ptr,
                 _dev.ptr(yy_cache), _dev.ptr(met_ws), met_ws.numel(), stream)
            e2 = torch.cuda.Event(enable_timing=True)
            e2.record()
        _dev.nvtx_push("flow")
        if sharded and cfg.method == "sinkhorn":
            shard_flow.flow_into(X, warm_f, warm_p, warm_valid, flow, fstat, state, it, flow_log,
                                 float(cfg.convergence_tol))
        elif sharded:
            shard_flow.flow_into(X, flow, fstat, state, it, flow_log, float(cfg.convergence_tol))
        elif cfg.method == "sinkhorn":
            call("fcb_sinkhorn_flow", prec, _dev.ptr(X), T, _dev.ptr(Yd), M, d, omega_fixed,
                 scfg.max_iters, scfg.tol, _dev.ptr(warm_f), _dev.ptr(warm_p),
                 _dev.ptr(warm_valid), _dev.ptr(flow), _dev.ptr(fstat), state_ptr, it,
                 _dev.ptr(flow_log), float(cfg.convergence_tol), _dev.ptr(flow_ws),
                 flow_ws.numel(), stream)
        else:
            call("fcb_stein_flow_full", prec, _dev.ptr(X), T, d, q.num_components,
                 _dev.ptr(gmm), bw_fixed, log_np1, _dev.ptr(flow), _dev.ptr(fstat), state_ptr,
                 it, _dev.ptr(flow_log), float(cfg.convergence_tol), _dev.ptr(flow_ws),
                 flow_ws.numel(), stream)
        _dev.nvtx_pop()
        e3 = torch.cuda.Event(enable_timing=True)
        e3.record()
        # state-independent Jacobians: the Riccati phase is computed once
        lqr_mode = 1 if (linear_model and it > 0) else 0
        _dev.nvtx_push("lqr")
        call("fcb_plan_update", spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(Sbuf[cur]),
             _dev.ptr(Ubuf[cur]), T, float(disc.dt), d, _dev.ptr(P), _dev.ptr(flow),
             _dev.ptr(Q), _dev.ptr(R), float(cfg.eta), _dev.ptr(clamp_d),
             _dev.ptr(Ubuf[1 - cur]), _dev.ptr(lqr_costs), state_ptr, it, lqr_mode,
             _dev.ptr(upd_ws), upd_ws.numel(), stream)
        _dev.nvtx_pop()
        e4 = torch.cuda.Event(enable_timing=True)
        e4.record()
        e_prev = e4
        marks.append((e0, e1, e2, e3, e4))
        if (it + 1) % poll_every != 0 and it + 1 < maxit:
            continue
        # asynchronous status snapshot; the host stays at most poll_lag
        # snapshots ahead of the device and stops queueing after a stop
        snap = ring[(it // poll_every) % len(ring)]
        snap.copy_(state, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        pending.append((it, ev, snap))
        stop = False
        while len(pending) > poll_lag:
            _k, evk, snapk = pending.popleft()
            evk.synchronize()
            if int(snapk[0]) != 0:
                stop = True
                break
        if stop:
            break

    status_host.copy_(state)
    torch.cuda.synchronize()
    st = status_host.numpy().copy()
    stop_kind, stage_code, fail_it, fail_idx, flows_used, updates = (int(v) for v in st[:6])

    def trajectory_of(k: int) -> Trajectory | None:
        if k < 0:
            return None
        return Trajectory(S=_dev.host(Sbuf[k & 1]).copy(), U=_dev.host(Ubuf[k & 1]).copy(),
                          dt=disc.dt)

    if stop_kind == 2:
        if stage_code == 1:
            raise PlanError("rollout", fail_it, trajectory_of(fail_it - 1),
                            RolloutDivergenceError(fail_idx))
        if stage_code == 2:
            worst = float(fstat[0].item())
            raise PlanError("flow", fail_it, trajectory_of(fail_it),
                            FlowError(flow_error_message(worst, cfg.sinkhorn.tol)))
        raise PlanError("lqr", fail_it, trajectory_of(fail_it), RiccatiDivergenceError(fail_idx))

    converged = stop_kind == 1
    iterations_used = flows_used
    log = _dev.host(flow_log[:iterations_used]).copy()
    costs = _dev.host(lqr_costs[:updates]).copy()

    # phase times over the iterations that actually ran
    t_flow = t_lqr = t_roll = 0.0
    for k, (e0, e1, e2, e3, e4) in enumerate(marks[:iterations_used]):
        t_roll += e0.elapsed_time(e1) * 1e-3
        t_flow += e2.elapsed_time(e3) * 1e-3
        if k < updates:
            t_lqr += e3.elapsed_time(e4) * 1e-3
    if fused_ran:  # device-side phase clocks of the persistent launch
        pn = phase_ns.cpu().numpy().astype(np.float64) * 1e-9
        t_roll += float(pn[0])
        t_flow += float(pn[1])
        t_lqr += float(pn[2])

    # final rollout on the last controls (optimizer.py:271-277)
    U_final = Ubuf[updates & 1]
    status = torch.empty(1, dtype=torch.int32, device=dev)
    ef0 = torch.cuda.Event(enable_timing=True)
    ef0.record()
    S_final = _dev.zeros((T + 1, n_s), device=dev)
    call("fcb_rollout", spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(s0), _dev.ptr(U_final),
         T, float(disc.dt), _dev.ptr(S_final), d, _dev.ptr(P), _dev.ptr(X), _dev.ptr(status),
         None, 0, rollout_method(T), _dev.ptr(roll_ws), stream)
    ef1 = torch.cuda.Event(enable_timing=True)
    ef1.record()
    ef1.synchronize()
    t_roll += ef0.elapsed_time(ef1) * 1e-3
    fstep = int(status.item())
    if fstep >= 0:
        raise PlanError("rollout", updates, trajectory_of(iterations_used - 1),
                        RolloutDivergenceError(fstep))
    trajectory = Trajectory(S=_dev.host(S_final).copy(), U=_dev.host(U_final).copy(), dt=disc.dt)

    metric_iters: list[int] = []
    metric_values: list[float] = []
    final_metric = None
    if want_metric:
        vals = _dev.host(metric_vals[:, 0])
        for it in range(iterations_used):
            if it % cfg.metric_interval == 0:
                metric_iters.append(it)
                metric_values.append(float(vals[it // cfg.metric_interval]))
        fm = _dev.empty((4,), device=dev)
        call("fcb_sinkhorn_divergence_cached", mprec, _dev.ptr(X), T, _dev.ptr(Ymd), Mm, d,
             _omega_arg(cfg.sinkhorn.omega), cfg.sinkhorn.max_iters, cfg.sinkhorn.tol,
             _dev.ptr(fm), None, _dev.ptr(yy_cache), _dev.ptr(met_ws), met_ws.numel(), stream)
        final_metric = float(fm[0].item())
        if not metric_iters or metric_iters[-1] != updates:
            metric_iters.append(updates)
            metric_values.append(final_metric)

    launches = lib.fcb_launch_count() - launches0
    result = PlanResult(
        trajectory=trajectory,
        converged=converged,
        iterations_used=iterations_used,
        flow_norms=log[:, 0].copy(),
        lqr_costs=costs,
        metric_iterations=tuple(metric_iters),
        metric_values=tuple(metric_values),
        phase_times=PhaseTimes(flow=t_flow, lqr=t_lqr, rollout=t_roll,
                               total=time.perf_counter() - t_begin),
        final_metric=final_metric,
    )
    return PlanRun(
        result=result,
        flow_log=log,
        precision=prec,
        pairs=_pair_count(cfg.method, log, T, M),
        launches=int(launches),
    )


# ---------------------------------------------------------------------------
# batched independent problems (BASELINE config 5)
# ---------------------------------------------------------------------------
def _batch_key(model: DynamicsModel, disc: Discretization, cfg: PlanConfig) -> tuple:
    """Everything but the seed, the start state and the targets must agree."""
    c = cfg
    return (device_model(model).model_id, model.state_dim, model.control_dim,
            model.workspace_dim, disc.num_steps, disc.dt, c.method, c.eta, c.max_iterations,
            c.convergence_tol, c.control_clamp, c.init_scale, c.metric_interval, c.q_weight,
            c.r_weight, c.sinkhorn, isinstance(c.initial_controls, str) and c.initial_controls)


def plan_batch_detailed(problems: list) -> list[PlanRun]:
    """Plan independent problems [(model, q, disc, cfg), ...] on this GPU.

    Each result follows plan() of that problem (optimizer.py:171-304).  When
    every problem is a built-in linear model with the same shapes and
    configuration (seeds, start states and targets may differ), the Sinkhorn
    method, no in-loop metric and point sets that fit on chip, the whole
    batch runs as ONE launch of the fused planner with one problem per CTA
    (fcb_plan_fused, batch > 1); otherwise the problems run one by one.  As in
    a loop over plan(), the first failing problem (in order) raises its
    PlanError.
    """
    if not problems:
        return []
    model, _q, disc, cfg = problems[0]
    key = _batch_key(model, disc, cfg)
    uniform = len(problems) > 1 and all(_batch_key(m, ds, c) == key for m, _, ds, c in problems)
    spec = device_model(model)
    T = disc.num_steps
    d = model.workspace_dim
    eligible = (uniform and cfg.method == "sinkhorn" and cfg.metric_interval == 0 and d == 2
                and cfg.max_iterations >= 1 and os.environ.get("FCB_FUSED", "1") != "0"
                and spec.model_id in (_lib.FCB_MODEL_SINGLE_INTEGRATOR_2D,
                                      _lib.FCB_MODEL_DOUBLE_INTEGRATOR_2D))
    targets = []
    if eligible:
        for m, q, ds, c in problems:
            if ds.s0.shape != (m.state_dim,):
                raise ValueError(f"s0 must have shape ({m.state_dim},), got {ds.s0.shape}")
            tg = q if isinstance(q, SamplePoints) else to_sample_based(
                q, T, [c.seed, STREAM_REFERENCE])
            targets.append(np.asarray(tg.points, dtype=np.float64))
        M = targets[0].shape[0]
        eligible = all(t.shape == (M, d) for t in targets)
    if eligible:
        prec = _precision.pick(cfg.sinkhorn.precision, T * max(T, M), cfg.sinkhorn.tol)
        eligible = prec == _lib.FCB_FP32
    if not eligible:
        return [plan_detailed(*p) for p in problems]

    B = len(problems)
    lib = _lib.load()
    dev = _dev.require_cuda()
    stream = _dev.stream()
    t_begin = time.perf_counter()
    n_s, m_c = model.state_dim, model.control_dim
    maxit = cfg.max_iterations
    weights = workspace_weights(model.project_matrix, m_c, cfg.q_weight, cfg.r_weight)
    clamp = cfg.control_clamp
    if clamp is not None and len(clamp) != m_c:
        raise ValueError(f"control_clamp needs {m_c} bounds, got {len(clamp)}")
    bounds = np.asarray(clamp, dtype=np.float64) if clamp is not None else None
    U0 = np.stack([initial_controls(c, m, T) for m, _, _, c in problems])
    if bounds is not None:
        np.clip(U0, -bounds, bounds, out=U0)
    s0 = _dev.f64(np.stack([ds.s0 for _, _, ds, _ in problems]), dev)
    Yd = _dev.f64(np.stack(targets), dev)
    Ubuf = [_dev.f64(U0, dev), _dev.zeros((B, T, m_c), device=dev)]
    Sbuf = [_dev.zeros((B, T + 1, n_s), device=dev), _dev.zeros((B, T + 1, n_s), device=dev)]
    X = _dev.zeros((B, T, d), device=dev)
    flow = _dev.zeros((B, T, d), device=dev)
    P = _dev.f64(model.project_matrix, dev)
    Q = _dev.f64(weights.Q, dev)
    R = _dev.f64(weights.R, dev)
    clamp_d = _dev.f64(bounds, dev) if bounds is not None else None
    prm = spec.device_params(dev)
    state = torch.zeros((B, 8), dtype=torch.int32, device=dev)
    flow_log = _dev.zeros((B, maxit, 4), device=dev)
    lqr_costs = _dev.zeros((B, maxit), device=dev)
    fstat = _dev.zeros((B, 8), device=dev)
    warm_f, warm_p = _dev.zeros((B, T), device=dev), _dev.zeros((B, T), device=dev)
    warm_valid = torch.zeros((B, 2), dtype=torch.int32, device=dev)
    phase_ns = torch.zeros((B, 3), dtype=torch.int64, device=dev)
    scfg = cfg.sinkhorn

    def call(name, *args):
        _lib.check(getattr(lib, name)(*args), name)

    # the stored Riccati phase: the built-in linear models' Jacobians are
    # state-independent, so one mode-0 update on scratch inputs computes it
    upd_ws = _dev.Workspace.get(lib.fcb_plan_update_workspace_bytes(n_s, m_c, T), "batch_upd")
    scratch_state = torch.zeros(8, dtype=torch.int32, device=dev)
    call("fcb_plan_update", spec.model_id, n_s, m_c, _dev.ptr(prm),
         _dev.ptr(_dev.zeros((T + 1, n_s), device=dev)), _dev.ptr(_dev.zeros((T, m_c), device=dev)),
         T, float(disc.dt), d, _dev.ptr(P), _dev.ptr(_dev.zeros((T, d), device=dev)), _dev.ptr(Q),
         _dev.ptr(R), float(cfg.eta), _dev.ptr(clamp_d),
         _dev.ptr(_dev.zeros((T, m_c), device=dev)), _dev.ptr(_dev.zeros((maxit,), device=dev)),
         _dev.ptr(scratch_state), 0, 0, _dev.ptr(upd_ws), upd_ws.numel(), stream)
    fws = _dev.Workspace.get(lib.fcb_plan_fused_workspace_bytes(B, T, M, d, m_c), "batch_fused")
    launches0 = lib.fcb_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = lib.fcb_plan_fused(
        spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(s0), _dev.ptr(Ubuf[0]),
        _dev.ptr(Ubuf[1]), _dev.ptr(Sbuf[0]), _dev.ptr(Sbuf[1]), T, float(disc.dt), d,
        _dev.ptr(P), _dev.ptr(X), _dev.ptr(flow), _dev.ptr(Q), _dev.ptr(R), float(cfg.eta),
        _dev.ptr(clamp_d), _dev.ptr(Yd), M, _omega_arg(scfg.omega), scfg.max_iters, scfg.tol,
        float(cfg.convergence_tol), _dev.ptr(warm_f), _dev.ptr(warm_p), _dev.ptr(warm_valid),
        _dev.ptr(fstat), _dev.ptr(state), _dev.ptr(flow_log), _dev.ptr(lqr_costs),
        _dev.ptr(phase_ns), 0, maxit, B, _dev.ptr(upd_ws), _dev.ptr(fws), fws.numel(), stream)
    if rc == _lib.FCB_ENOTSUP:
        return [plan_detailed(*p) for p in problems]
    _lib.check(rc, "fcb_plan_fused")
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    e1.synchronize()
    st_all = state.cpu().numpy()
    logs = flow_log.cpu().numpy()
    costs_all = lqr_costs.cpu().numpy()
    pn_all = phase_ns.cpu().numpy().astype(np.float64) * 1e-9
    fst = fstat.cpu().numpy()
    # final rollouts on the last controls (optimizer.py:271-277): the B
    # single-warp rollouts are independent, so they run concurrently on side
    # streams with one synchronisation and bulk copies for the whole batch
    S_fin = _dev.zeros((B, T + 1, n_s), device=dev)
    X_fin = _dev.zeros((B, T, d), device=dev)
    fin_status = torch.full((B,), -1, dtype=torch.int32, device=dev)
    method = rollout_method(T)
    side = [torch.cuda.Stream(device=dev) for _ in range(min(B, 16))]
    nws = lib.fcb_rollout_workspace_bytes(n_s, T)
    roll_ws = [_dev.Workspace.get(nws, f"batch_roll{k}") for k in range(len(side))]
    ready = torch.cuda.Event()
    ready.record()  # the buffers' fills above are on the current stream
    for sk in side:
        sk.wait_event(ready)
    for b in range(B):
        if int(st_all[b, 0]) == 2:
            continue
        k = b % len(side)
        call("fcb_rollout", spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(s0[b]),
             _dev.ptr(Ubuf[int(st_all[b, 5]) & 1][b]), T, float(disc.dt), _dev.ptr(S_fin[b]), d,
             _dev.ptr(P), _dev.ptr(X_fin[b]), _dev.ptr(fin_status[b:b + 1]), None, 0, method,
             _dev.ptr(roll_ws[k]), side[k].cuda_stream)
    for sk in side:
        sk.synchronize()
    S_fin_h = S_fin.cpu().numpy()
    U_h = [Ubuf[0].cpu().numpy(), Ubuf[1].cpu().numpy()]
    fin_h = fin_status.cpu().numpy()
    runs: list[PlanRun] = []
    for b in range(B):
        stop_kind, stage_code, fail_it, fail_idx, flows_used, updates = (
            int(v) for v in st_all[b, :6])

        def trajectory_of(k: int, b=b) -> Trajectory | None:
            if k < 0:
                return None
            return Trajectory(S=_dev.host(Sbuf[k & 1][b]).copy(),
                              U=_dev.host(Ubuf[k & 1][b]).copy(), dt=disc.dt)

        if stop_kind == 2:
            if stage_code == 1:
                raise PlanError("rollout", fail_it, trajectory_of(fail_it - 1),
                                RolloutDivergenceError(fail_idx))
            if stage_code == 2:
                raise PlanError("flow", fail_it, trajectory_of(fail_it),
                                FlowError(flow_error_message(float(fst[b, 0]), scfg.tol)))
            raise PlanError("lqr", fail_it, trajectory_of(fail_it),
                            RiccatiDivergenceError(fail_idx))
        fstep = int(fin_h[b])
        if fstep >= 0:
            raise PlanError("rollout", updates, trajectory_of(flows_used - 1),
                            RolloutDivergenceError(fstep))
        log = logs[b, :flows_used].copy()
        result = PlanResult(
            trajectory=Trajectory(S=S_fin_h[b].copy(), U=U_h[updates & 1][b].copy(),
                                  dt=disc.dt),
            converged=stop_kind == 1,
            iterations_used=flows_used,
            flow_norms=log[:, 0].copy(),
            lqr_costs=costs_all[b, :updates].copy(),
            metric_iterations=(),
            metric_values=(),
            phase_times=PhaseTimes(flow=float(pn_all[b, 1]), lqr=float(pn_all[b, 2]),
                                   rollout=float(pn_all[b, 0]),
                                   total=time.perf_counter() - t_begin),
            final_metric=None,
        )
        runs.append(PlanRun(result=result, flow_log=log, precision=prec,
                            pairs=_pair_count(cfg.method, log, T, M),
                            launches=int(lib.fcb_launch_count() - launches0)))
    return runs


def plan_batch(problems: list) -> list[PlanResult]:
    """plan() of every problem (batched on the device when they share a shape)."""
    return [r.result for r in plan_batch_detailed(problems)]
