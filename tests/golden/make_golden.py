"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--long]

It imports `flowcover` read-only from /root/reference/pkg/src and writes
small .npz fixtures next to this file.  tests/test_oracle_golden.py pins the
oracle against them; the GPU parity tests compare the CUDA path against them.
--long additionally runs BASELINE config 2 in full (200 outer iterations,
~5 min on 8 cores) for the end-to-end trajectory/coverage target.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("FLOWCOVER_WORKERS", str(os.cpu_count() or 1))

import flowcover as fc  # noqa: E402
from flowcover.seeding import STREAM_METRIC, STREAM_REFERENCE  # noqa: E402
from flowcover.sinkhorn import SinkhornWarmState  # noqa: E402


def save(name: str, **arrays) -> None:
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1024:.1f} KiB)")


def random_pair(seed, n, m, dim):
    rng = np.random.default_rng(seed)
    return rng.random((n, dim)), rng.random((m, dim))


def double_integrator_2d():
    A = np.zeros((4, 4))
    A[0, 2] = A[1, 3] = 1.0
    B = np.zeros((4, 2))
    B[2, 0] = B[3, 1] = 1.0
    P = np.zeros((2, 4))
    P[0, 0] = P[1, 1] = 1.0
    return fc.DynamicsModel(
        name="double_integrator_2d", state_dim=4, control_dim=2, workspace_dim=2,
        state_names=("x", "y", "vx", "vy"), control_names=("ax", "ay"),
        f=lambda s, u: np.array([s[2], s[3], u[0], u[1]]),
        jacobian_A=lambda s, u: A.copy(), jacobian_B=lambda s, u: B.copy(), project_matrix=P,
    )


# ---------------------------------------------------------------------------
def gen_ot():
    cases = [
        # seed, n, m, dim, omega, max_iters, tol
        (0, 8, 7, 2, 0.05, 50_000, 1e-10),
        (1, 40, 55, 3, "auto", 1000, 1e-6),
        (2, 64, 50, 1, 0.1, 50_000, 1e-10),
        (3, 200, 300, 2, "auto", 1000, 1e-6),
        (4, 12, 15, 2, 0.01, 3, 1e-14),  # budget-limited, unconverged
        (5, 1500, 2500, 2, "auto", 1000, 1e-6),
        (6, 700, 900, 3, "auto", 1000, 1e-6),
    ]
    out = {}
    for k, (seed, n, m, dim, omega, mi, tol) in enumerate(cases):
        X, Y = random_pair(seed, n, m, dim)
        if seed == 4:
            Y = Y + 10.0
        cfg = fc.SinkhornConfig(omega=omega, max_iters=mi, tol=tol)
        sol = fc.entropic_ot(X, Y, cfg)
        out.update({
            f"c{k}_X": X, f"c{k}_Y": Y,
            f"c{k}_cfg": np.array([0.0 if omega == "auto" else omega, mi, tol]),
            f"c{k}_f": sol.f, f"c{k}_g": sol.g,
            f"c{k}_scal": np.array([sol.cost, sol.iters_used, float(sol.converged),
                                    sol.marginal_error, sol.omega]),
        })
        if n * m <= 4000:
            out[f"c{k}_plan"] = sol.plan()
    # single sweeps of _lse_rows on a larger instance (per-sweep parity)
    from flowcover.sinkhorn import _lse_rows, _pairwise_sq

    X, Y = random_pair(11, 3000, 5000, 2)
    pot = np.random.default_rng(12).normal(scale=0.01, size=5000)
    C = _pairwise_sq(X, Y)
    L = np.empty(3000)
    _lse_rows(C, pot, 0.02, L, 256, 1)
    out.update(sweep_X=X, sweep_Y=Y, sweep_pot=pot, sweep_omega=np.array(0.02), sweep_L=L)
    out["ncases"] = np.array(len(cases))
    save("ot_cases.npz", **out)


def gen_flow_and_divergence():
    out = {}
    cases = [
        (6, 30, 30, 2, 0.05, 50_000, 1e-10),
        (8, 150, 120, 2, 0.05, 1000, 1e-10),
        (9, 500, 2000, 2, "auto", 1000, 1e-6),
        (10, 400, 300, 3, "auto", 1000, 1e-6),
        (13, 2000, 10_000, 2, "auto", 1000, 1e-6),
    ]
    for k, (seed, n, m, dim, omega, mi, tol) in enumerate(cases):
        X, Y = random_pair(seed, n, m, dim)
        cfg = fc.SinkhornConfig(omega=omega, max_iters=mi, tol=tol)
        warm = SinkhornWarmState()
        first = fc.sinkhorn_flow(X, fc.SamplePoints(points=Y), cfg, warm=warm)
        # second call from the warm state at a perturbed X (a planner step)
        X2 = X + 1e-3 * first.a / max(np.abs(first.a).max(), 1e-30)
        second = fc.sinkhorn_flow(X2, fc.SamplePoints(points=Y), cfg, warm=warm)
        out.update({
            f"c{k}_X": X, f"c{k}_Y": Y, f"c{k}_X2": X2,
            f"c{k}_cfg": np.array([0.0 if omega == "auto" else omega, mi, tol]),
            f"c{k}_a": first.a, f"c{k}_a2": second.a,
            f"c{k}_scal": np.array([float(first.converged), first.marginal_error,
                                    float(second.converged), second.marginal_error]),
            f"c{k}_warm_f": warm.f, f"c{k}_warm_p": warm.p,
        })
        if n * m <= 1_000_000:
            out[f"c{k}_div"] = np.array(fc.sinkhorn_divergence(X, Y, cfg))
    out["ncases"] = np.array(len(cases))
    save("flow_cases.npz", **out)


def gen_stein():
    out = {}
    q2 = fc.benchmark_mixture(2)
    q3 = fc.benchmark_mixture(3)
    cases = [
        (1, 40, 2, "median"),
        (2, 41, 2, "median"),
        (3, 300, 2, 0.2),
        (4, 500, 2, "median"),
        (5, 257, 3, "median"),
        (6, 1000, 2, "median"),
        (7, 64, 1, 0.5),
    ]
    for k, (seed, n, dim, bw) in enumerate(cases):
        rng = np.random.default_rng(seed)
        pts = rng.normal(loc=0.5, scale=0.3, size=(n, dim))
        if dim == 1:
            q = fc.GaussianMixture(weights=np.array([1.0]), means=np.zeros((1, 1)),
                                   covariances=np.eye(1)[None])
        else:
            q = q2 if dim == 2 else q3
        res = fc.stein_flow(pts, q, fc.SteinConfig(bandwidth=bw))
        out.update({
            f"c{k}_X": pts, f"c{k}_dim": np.array(dim),
            f"c{k}_bw": np.array(-1.0 if bw == "median" else bw),
            f"c{k}_a": res.a, f"c{k}_h": np.array(res.bandwidth),
            f"c{k}_med_h": np.array(fc.median_bandwidth(pts)),
        })
    out["ncases"] = np.array(len(cases))
    # mixture score / log density
    rng = np.random.default_rng(8)
    w = rng.random(3)
    w /= w.sum()
    covs = []
    for _ in range(3):
        M = rng.normal(size=(2, 2))
        covs.append(0.05 * np.eye(2) + 0.3 * M @ M.T)
    qr = fc.GaussianMixture(weights=w, means=rng.uniform(-1, 1, (3, 2)), covariances=np.stack(covs))
    Xs = rng.uniform(-2, 2, (500, 2))
    X3 = rng.uniform(0, 1, (300, 3))
    out.update(
        gmm_w=qr.weights, gmm_mu=qr.means, gmm_cov=qr.covariances, gmm_X=Xs,
        gmm_score=qr.score(Xs), gmm_logd=qr.log_density(Xs),
        gmm3_X=X3, gmm3_score=q3.score(X3), gmm3_logd=q3.log_density(X3),
        sample2=q2.sample(1000, [0, STREAM_METRIC]),
    )
    save("stein_cases.npz", **out)


def gen_dynamics_lqr():
    out = {}
    models = {
        "single_integrator_2d": fc.single_integrator_2d(),
        "diff_drive": fc.differential_drive(),
        "aircraft_3d": fc.aircraft_3d(),
        "double_integrator_2d": double_integrator_2d(),
    }
    for k, (name, m) in enumerate(models.items()):
        rng = np.random.default_rng(100 + k)
        T = 300
        U = rng.normal(scale=0.4, size=(T, m.control_dim))
        s0 = fc.default_start(m) if name != "double_integrator_2d" else np.array([0.1, 0.1, 0, 0])
        S = fc.rollout(m, s0, U, 0.05)
        sys_ = fc.linearize_along(m, S, U, 0.05)
        out.update({f"{name}_U": U, f"{name}_s0": s0, f"{name}_S": S,
                    f"{name}_A": sys_.A, f"{name}_B": sys_.B})
    # LQR: random systems (test_lqr.py:19-28 style)
    for T in (1, 2, 3, 5, 10, 200, 2000):
        rng = np.random.default_rng(100 + T)
        n, m = 3, 2
        A = 0.3 * rng.normal(size=(T, n, n))
        B = rng.normal(size=(T, n, m))
        C = rng.normal(size=(n, n))
        D = rng.normal(size=(m, m))
        w = fc.LqrWeights(Q=C.T @ C, R=D.T @ D + 0.1 * np.eye(m))
        a = rng.normal(size=(T, n))
        sol = fc.solve_flow_lqr(fc.LtvSystem(A=A, B=B, dt=0.05), a, w)
        out.update({f"lqr{T}_A": A, f"lqr{T}_B": B, f"lqr{T}_Q": w.Q, f"lqr{T}_R": w.R,
                    f"lqr{T}_a": a, f"lqr{T}_v": sol.v_star, f"lqr{T}_z": sol.z,
                    f"lqr{T}_K": sol.K, f"lqr{T}_d": sol.d, f"lqr{T}_cost": np.array(sol.cost)})
    save("dyn_lqr_cases.npz", **out)


def _record_flows(fn_name):
    """Wrap the reference flow so per-iteration (X, flow) pairs are recorded."""
    import flowcover.optimizer as opt

    records = []
    orig = getattr(opt, fn_name)

    def wrapped(*args, **kwargs):
        res = orig(*args, **kwargs)
        records.append((np.array(args[0], copy=True), res.a.copy()))
        return res

    setattr(opt, fn_name, wrapped)
    return records, lambda: setattr(opt, fn_name, orig)


def run_plan(tag, model, q, disc, cfg, record=False):
    fn = "sinkhorn_flow" if cfg.method == "sinkhorn" else "stein_flow_on_trajectory"
    recs, restore = _record_flows(fn) if record else ([], lambda: None)
    t0 = time.perf_counter()
    try:
        res = fc.plan(model, q, disc, cfg)
    finally:
        restore()
    dt = time.perf_counter() - t0
    print(f"  {tag}: {dt:.1f}s, {res.iterations_used} iterations")
    out = {
        f"{tag}_S": res.trajectory.S, f"{tag}_U": res.trajectory.U,
        f"{tag}_flow_norms": res.flow_norms, f"{tag}_lqr_costs": res.lqr_costs,
        f"{tag}_metric_it": np.array(res.metric_iterations, dtype=np.int64),
        f"{tag}_metric_val": np.array(res.metric_values, dtype=np.float64),
        f"{tag}_final_metric": np.array(np.nan if res.final_metric is None else res.final_metric),
        f"{tag}_meta": np.array([res.iterations_used, float(res.converged), dt]),
    }
    for i, (Xk, ak) in enumerate(recs[:3]):
        out[f"{tag}_rec{i}_X"] = Xk if cfg.method == "sinkhorn" else model.project_states(Xk[1:])
        out[f"{tag}_rec{i}_a"] = ak
    return out


def gen_plans(long: bool):
    out = {}
    di = double_integrator_2d()
    q2 = fc.benchmark_mixture(2)
    # config-1 (BASELINE configs[0]): DI, SVGD median, T=500, 100 it, eta=0.1, metric vs 1000
    out.update(run_plan(
        "cfg1", di, q2, fc.Discretization(0.05, 500, np.array([0.1, 0.1, 0.0, 0.0])),
        fc.PlanConfig(method="stein", eta=0.1, max_iterations=100, convergence_tol=0.0,
                      metric_interval=25, metric_samples=1000, seed=0), record=True))
    # config-2 shape (T=2000, M=1e4) for 3 outer iterations (per-iteration flows)
    targets = fc.SamplePoints(q2.sample(10_000, [0, STREAM_REFERENCE]))
    out.update(run_plan(
        "cfg2s", di, targets, fc.Discretization(0.05, 2000, np.array([0.1, 0.1, 0.0, 0.0])),
        fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=3, convergence_tol=0.0,
                      metric_interval=0, seed=0), record=True))
    # small planner cases with metric cadence
    out.update(run_plan(
        "si_sk", fc.single_integrator_2d(), q2, fc.Discretization(0.05, 200, np.array([0.1, 0.1])),
        fc.PlanConfig(method="sinkhorn", eta=30.0, max_iterations=20, convergence_tol=0.0,
                      metric_interval=5, metric_samples=300, seed=0)))
    out.update(run_plan(
        "dd_st", fc.differential_drive(), q2, fc.Discretization(0.05, 300, np.array([0.1, 0.1, 0.0])),
        fc.PlanConfig(method="stein", eta=0.1, max_iterations=15, convergence_tol=0.0,
                      metric_interval=5, metric_samples=300, seed=4)))
    q3 = fc.benchmark_mixture(3)
    out.update(run_plan(
        "ac_sk", fc.aircraft_3d(), q3,
        fc.Discretization(0.05, 300, fc.default_start(fc.aircraft_3d())),
        fc.PlanConfig(method="sinkhorn", eta=45.0, max_iterations=10, convergence_tol=0.0,
                      metric_interval=0, seed=0)))
    save("plan_cases.npz", **out)
    if long:
        res = run_plan(
            "cfg2", di, targets, fc.Discretization(0.05, 2000, np.array([0.1, 0.1, 0.0, 0.0])),
            fc.PlanConfig(method="sinkhorn", eta=300.0, max_iterations=200, convergence_tol=0.0,
                          metric_interval=0, seed=0))
        draws = q2.sample(10_000, [0, STREAM_METRIC])
        res["cfg2_coverage"] = np.array(
            fc.coverage_metric(res["cfg2_S"], di, draws, fc.SinkhornConfig()))
        save("plan_cfg2_full.npz", **res)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--long", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    jobs = dict(ot=gen_ot, flow=gen_flow_and_divergence, stein=gen_stein, dyn=gen_dynamics_lqr,
                plan=lambda: gen_plans(args.long))
    for name, fn in jobs.items():
        if args.only and name not in args.only.split(","):
            continue
        t0 = time.perf_counter()
        fn()
        print(f"[{name}] {time.perf_counter() - t0:.1f}s")
