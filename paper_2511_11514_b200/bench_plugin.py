"""B200 planners for the reference's benchmark harness (bench.py:158-209).

The reference times its planners through closures `run(horizon, workers) ->
PlannerRun` built by `standard_planners(spec)` and writes one CSV row per
(method, horizon, repeat) (bench.py:221-309).  `b200_planners(spec)` builds
the same closures over this package's device planner, so the reference's own
harness, CSV schema and alpha-fit tooling (scaling figures) run unchanged
with GPU curves next to the CPU ones:

    # flowcover/bench.py, in standard_planners(), before `return`:
    if os.environ.get("FLOWCOVER_BACKEND") == "b200":
        import paper_2511_11514_b200.bench_plugin as b200
        planners.update(b200.b200_planners(spec, PlannerRun))

Planner names are "b200-stein" and "b200-sinkhorn"; configuration follows the
reference's study defaults (STUDY_ITERATIONS = 20 fixed iterations, fixed
Stein bandwidth 0.02, eta 0.1, metric off during timing; bench.py:42-44,
:169-178).  `workers` is accepted and ignored, as the device path has no
thread pool.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Any, Callable

from .dynamics import Discretization, Trajectory, default_start, get_model
from .optimizer import PlanConfig, plan
from .reference import benchmark_mixture
from .stein import SteinConfig

STUDY_ITERATIONS = 20     # bench.py:42
STUDY_BANDWIDTH = 0.02    # bench.py:43


@dataclass(frozen=True)
class PlannerRun:
    """Mirror of the reference's bench.PlannerRun (bench.py:148-155)."""

    trajectory: Trajectory
    t_flow: float
    t_lqr: float
    t_rollout: float


def b200_planners(spec: Any, planner_run: Callable[..., Any] | None = None,
                  reference_names: bool = False) -> dict[str, Callable]:
    """Planner closures for a reference BenchSpec (duck-typed: model, dt, seed, plan).

    planner_run: the harness's PlannerRun class (defaults to this module's
    mirror), so the rows it writes are the reference's own type.
    reference_names: key the closures "stein" / "sinkhorn" -- the method names
    BenchSpec validates (bench.py:67-69) -- so `run_bench(spec, planners=...)`
    times the device planners under the stock spec; default keys are
    "b200-stein" / "b200-sinkhorn" for merging into standard_planners().
    """
    make_run = planner_run or PlannerRun
    model = get_model(spec.model)
    q = benchmark_mixture(model.workspace_dim)
    s0 = default_start(model)
    plan_base = getattr(spec, "plan", None)
    if plan_base is None or not isinstance(plan_base, PlanConfig):
        base = PlanConfig(eta=0.1, max_iterations=STUDY_ITERATIONS, convergence_tol=0.0,
                          stein=SteinConfig(bandwidth=STUDY_BANDWIDTH))
        if plan_base is not None:  # a reference PlanConfig: carry its scalar fields over
            base = replace(base, eta=plan_base.eta, max_iterations=plan_base.max_iterations,
                           convergence_tol=plan_base.convergence_tol)
        plan_base = base
    base_cfg = replace(plan_base, seed=spec.seed, metric_interval=0)

    def flow_planner(method: str) -> Callable:
        def run(horizon: int, workers: int) -> Any:
            cfg = replace(base_cfg, method=method, workers=workers)
            res = plan(model, q, Discretization(spec.dt, horizon, s0), cfg)
            t = res.phase_times
            return make_run(res.trajectory, t.flow, t.lqr, t.rollout)

        return run

    prefix = "" if reference_names else "b200-"
    return {f"{prefix}stein": flow_planner("stein"), f"{prefix}sinkhorn": flow_planner("sinkhorn")}
