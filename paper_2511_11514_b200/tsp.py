"""The TSP-waypoint baseline (tsp.py), on the GPU.

Drop-in for the reference's tsp.py: the same `Tour`, `tour_length`,
`build_tour(points, seed, budget)`, `resample_arclength`, `track_waypoints`,
`BaselineConfig` / `BaselineResult` and `baseline_plan` signatures and results.

  * Tours (tsp.py:30-147): the nearest-neighbour order and the
    first-improving 2-opt search run in `fcb_tsp_tours` (csrc/tsp.cu), one CTA
    per problem with the point set in shared memory; `build_tours` plans many
    problems in one launch (BASELINE config 5 compares 4096 planned problems
    against 4096 TSP baselines).  Only the start index is drawn on the host,
    from the reference's stream [seed, 4].
  * Tracking (tsp.py:150-273): the path is resampled by arc length and lifted
    to a start state and control guess on the host (O(T) numpy, as the
    reference); the iterated time-varying LQR then runs on the device as the
    planner's own update step -- per round one rollout (`fcb_rollout`), the
    tracking error ref - P s_k as the flow, and `fcb_plan_update` with step 1
    and no clamp (linearise, Riccati, affine phase, U += v*) -- with no host
    round trip until the final rollout.

The baseline is what the flow planners are compared with, not the product; it
lives here so the comparison can be run at config-5 scale.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import numpy.typing as npt
import torch

from . import _dev, _lib
from .dynamics import (
    Discretization,
    DynamicsModel,
    RolloutDivergenceError,
    Trajectory,
    device_model,
    rollout_method,
)
from .lqr import RiccatiDivergenceError, workspace_weights
from .optimizer import PhaseTimes
from .seeding import STREAM_REFERENCE, STREAM_TOUR, rng_stream

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


# ---------------------------------------------------------------------------
# tracking stage (tsp.py:150-316)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class BaselineConfig:
    """tsp.py:44-57: tour seed, 2-opt budget (0: 10 n), tracking rounds, weights."""

    seed: int = 0
    budget: int = 0
    track_iterations: int = 10
    q_weight: float = 1.0
    r_weight: float = 0.1

    def __post_init__(self) -> None:
        if self.budget < 0:
            raise ValueError(f"budget must be >= 0 (0 means automatic), got {self.budget}")
        if self.track_iterations < 1:
            raise ValueError(f"track_iterations must be >= 1, got {self.track_iterations}")


@dataclass(frozen=True)
class BaselineResult:
    trajectory: Trajectory
    tour: Tour
    waypoints: npt.NDArray[np.float64]
    phase_times: PhaseTimes


def resample_arclength(points, count: int) -> npt.NDArray[np.float64]:
    """`count` points spaced uniformly in arc length along the ordered polyline
    (tsp.py:150-167); repeated consecutive points are dropped first."""
    P = np.asarray(points, dtype=np.float64)
    if P.ndim != 2 or len(P) < 1:
        raise ValueError("points must be a nonempty (n, d) array")
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    if len(P) > 1:
        steps = np.sqrt(((P[1:] - P[:-1]) ** 2).sum(axis=1))
        P = P[np.concatenate(([True], steps > 0.0))]
    if len(P) == 1:
        return np.repeat(P[:1], count, axis=0)
    s = np.concatenate(([0.0], np.cumsum(np.sqrt(((P[1:] - P[:-1]) ** 2).sum(axis=1)))))
    at = np.linspace(0.0, s[-1], count)
    return np.stack([np.interp(at, s, P[:, k]) for k in range(P.shape[1])], axis=1)


def _wrap(a):
    return (a + np.pi) % (2.0 * np.pi) - np.pi


def _headings(seg):
    """Segment lengths and, per segment, the latest segment at or before it
    with nonzero length (-1 before the first), so zero-length segments keep the
    previous heading (tsp.py:174-180)."""
    lens = np.sqrt((seg ** 2).sum(axis=1))
    last = np.maximum.accumulate(np.where(lens > 0.0, np.arange(len(seg)), -1))
    return lens, last


def _lift_reference(model: DynamicsModel, R, dt: float):
    """Start state and control guess following the resampled path R (T+1
    points) for the models the reference lifts (tsp.py:183-225)."""
    T = len(R) - 1
    seg = R[1:] - R[:-1]
    lens, last = _headings(seg)
    idx = np.clip(last, 0, None)
    known = last >= 0
    speed = lens / dt
    if model.name == "single_integrator_2d":
        return R[0].copy(), seg / dt
    if model.name == "diff_drive":
        psi = np.where(known, np.arctan2(seg[:, 1], seg[:, 0])[idx], 0.0)
        U = np.zeros((T, 2))
        U[:, 0] = speed
        U[:-1, 1] = _wrap(np.diff(psi)) / dt
        return np.array([R[0, 0], R[0, 1], psi[0]]), U
    if model.name == "aircraft_3d":
        psi = np.where(known, np.arctan2(seg[:, 1], seg[:, 0])[idx], 0.0)
        gam = np.where(known, np.arctan2(seg[:, 2], np.sqrt((seg[:, :2] ** 2).sum(axis=1)))[idx],
                       0.0)
        U = np.zeros((T, 3))
        U[:-1, 0] = _wrap(np.diff(psi)) / dt
        U[:-1, 1] = np.diff(gam) / dt
        U[:-1, 2] = np.diff(speed) / dt
        return np.array([R[0, 0], R[0, 1], R[0, 2], psi[0], gam[0], speed[0]]), U
    raise ValueError(f"no reference lift is defined for model {model.name!r}")


def track_waypoints(model: DynamicsModel, waypoints, T: int, dt: float, iterations: int = 10,
                    q_weight: float = 1.0, r_weight: float = 0.1,
                    timings: dict | None = None):
    """Iterated time-varying LQR tracking of an ordered waypoint path
    (tsp.py:228-273); returns the tracked (S, U) as host arrays."""
    W = np.asarray(waypoints, dtype=np.float64)
    if len(W) < 2:
        raise ValueError("need at least two waypoints")
    if T < 1:
        raise ValueError(f"T must be >= 1, got {T}")
    R = resample_arclength(W, T + 1)
    s0, U0 = _lift_reference(model, R, dt)
    w = workspace_weights(model.project_matrix, model.control_dim, q_weight, r_weight)
    spec = device_model(model)
    linear = spec.model_id in (_lib.FCB_MODEL_SINGLE_INTEGRATOR_2D,
                               _lib.FCB_MODEL_DOUBLE_INTEGRATOR_2D, _lib.FCB_MODEL_LTI)
    n_s, m_c, d = model.state_dim, model.control_dim, model.workspace_dim
    lib = _lib.load()
    dev = _dev.require_cuda()
    st = _dev.stream()
    ref = _dev.f64(R[1:], dev)
    s0d, P = _dev.f64(s0, dev), _dev.f64(model.project_matrix, dev)
    Q, Rw = _dev.f64(w.Q, dev), _dev.f64(w.R, dev)
    prm = spec.device_params(dev)
    Ub = [_dev.f64(U0, dev), _dev.zeros((T, m_c), device=dev)]
    S = _dev.zeros((T + 1, n_s), device=dev)
    X = _dev.zeros((T, d), device=dev)
    err = _dev.zeros((T, d), device=dev)
    costs = _dev.zeros((iterations,), device=dev)
    state = torch.zeros(8, dtype=torch.int32, device=dev)
    roll_ws = _dev.Workspace.get(lib.fcb_rollout_workspace_bytes(n_s, T), "track_roll")
    upd_ws = _dev.Workspace.get(lib.fcb_plan_update_workspace_bytes(n_s, m_c, T), "track_upd")
    # tracking rounds: the parallel-in-time rollout (as plan()'s loop); the
    # returned trajectory: the final rollout's method (sequential, bit-exact
    # with numpy for polynomial models, up to SEQUENTIAL_ROLLOUT_MAX_T)
    method_final = rollout_method(T)

    def call(name, *args):
        _lib.check(getattr(lib, name)(*args), name)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * iterations + 2)]
    for it in range(iterations):
        ev[2 * it].record()
        call("fcb_rollout", spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(s0d),
             _dev.ptr(Ub[it & 1]), T, float(dt), _dev.ptr(S), d, _dev.ptr(P), _dev.ptr(X), None,
             _dev.ptr(state), it, 1, _dev.ptr(roll_ws), st)
        ev[2 * it + 1].record()
        torch.sub(ref, X, out=err)  # the tracking error is the flow the update steers by
        call("fcb_plan_update", spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(S),
             _dev.ptr(Ub[it & 1]), T, float(dt), d, _dev.ptr(P), _dev.ptr(err), _dev.ptr(Q),
             _dev.ptr(Rw), 1.0, None, _dev.ptr(Ub[1 - (it & 1)]), _dev.ptr(costs),
             _dev.ptr(state), it, 1 if (linear and it > 0) else 0, _dev.ptr(upd_ws),
             upd_ws.numel(), st)
    U_fin = Ub[iterations & 1]
    status = torch.empty(1, dtype=torch.int32, device=dev)
    ev[2 * iterations].record()
    call("fcb_rollout", spec.model_id, n_s, m_c, _dev.ptr(prm), _dev.ptr(s0d), _dev.ptr(U_fin),
         T, float(dt), _dev.ptr(S), d, _dev.ptr(P), _dev.ptr(X), _dev.ptr(status), None, 0,
         method_final, _dev.ptr(roll_ws), st)
    ev[2 * iterations + 1].record()
    ev[-1].synchronize()
    code = state.cpu().numpy()
    if code[0] == 2:  # a tracking round failed: what the reference raises there
        if code[1] == 1:
            raise RolloutDivergenceError(int(code[3]))
        raise RiccatiDivergenceError(int(code[3]))
    step = int(status.item())
    if step >= 0:
        raise RolloutDivergenceError(step)
    if timings is not None:
        t_roll = sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(iterations + 1)) * 1e-3
        t_lqr = sum(ev[2 * k + 1].elapsed_time(ev[2 * k + 2]) for k in range(iterations)) * 1e-3
        timings["lqr"] = timings.get("lqr", 0.0) + t_lqr
        timings["rollout"] = timings.get("rollout", 0.0) + t_roll
    return _dev.host(S).copy(), _dev.host(U_fin).copy()


def baseline_plan(model: DynamicsModel, q, disc: Discretization,
                  cfg: BaselineConfig = BaselineConfig()) -> BaselineResult:
    """Targets, tour, resampled path, tracking (tsp.py:276-316).  The tracked
    trajectory starts on the path, not at disc.s0, as in the reference."""
    T = disc.num_steps
    points = q.sample(T, [cfg.seed, STREAM_REFERENCE])
    t_begin = time.perf_counter()
    t0 = time.perf_counter()
    tour = build_tour(points, cfg.seed, cfg.budget if cfg.budget else None)
    t_tour = time.perf_counter() - t0
    timings: dict = {}
    S, U = track_waypoints(model, points[tour.order], T, disc.dt, cfg.track_iterations,
                           cfg.q_weight, cfg.r_weight, timings)
    return BaselineResult(
        trajectory=Trajectory(S=S, U=U, dt=disc.dt),
        tour=tour,
        waypoints=points,
        phase_times=PhaseTimes(flow=t_tour, lqr=timings["lqr"], rollout=timings["rollout"],
                               total=time.perf_counter() - t_begin),
    )


def baseline_plans(model: DynamicsModel, q, disc: Discretization,
                   cfgs) -> list[BaselineResult]:
    """baseline_plan for many configurations (config 5: one per problem seed);
    equal to [baseline_plan(model, q, disc, c) for c in cfgs].  The tours of
    all problems are built in one launch (one CTA each), then every path is
    tracked.  The reference has no batch API; its callers loop."""
    cfgs = list(cfgs)
    if not cfgs:
        return []
    T = disc.num_steps
    t_begin = time.perf_counter()
    pts = [q.sample(T, [c.seed, STREAM_REFERENCE]) for c in cfgs]
    t0 = time.perf_counter()
    tours: list = [None] * len(cfgs)
    by_budget: dict = {}
    for k, c in enumerate(cfgs):
        by_budget.setdefault(c.budget if c.budget else 10 * T, []).append(k)
    for ks in by_budget.values():
        built = build_tours([(pts[k], cfgs[k].seed, cfgs[k].budget or None) for k in ks])
        for k, tour in zip(ks, built):
            tours[k] = tour
    t_tour = (time.perf_counter() - t0) / len(cfgs)
    out = []
    for k, c in enumerate(cfgs):
        timings: dict = {}
        S, U = track_waypoints(model, pts[k][tours[k].order], T, disc.dt, c.track_iterations,
                               c.q_weight, c.r_weight, timings)
        out.append(BaselineResult(
            trajectory=Trajectory(S=S, U=U, dt=disc.dt), tour=tours[k], waypoints=pts[k],
            phase_times=PhaseTimes(flow=t_tour, lqr=timings["lqr"], rollout=timings["rollout"],
                                   total=(time.perf_counter() - t_begin) / len(cfgs))))
    return out
