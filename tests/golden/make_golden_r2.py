"""Golden vectors for the fp32 paths of BASELINE configs 3-5 (round 2).

Run in the build container (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_r2.py [--only plans,large,batch]

Two sources, both pinned to the reference:

  plans  -- the UNMODIFIED reference (imported read-only from
            /root/reference/pkg/src) runs short plans at sizes where the
            device's precision="auto" picks the fp32 kernels (>= 2^20 pairs
            per sweep): diff_drive + Sinkhorn and aircraft_3d + Sinkhorn
            (T=800, M=2000), aircraft_3d + SVGD (T=1100, median h), plus the
            per-iteration (X, flow) pairs of their first iterations and the
            final coverage metric.  -> plan_fp32_cases.npz
  batch  -- the reference plans three BASELINE config-5 problems
            (single_integrator_2d, Sinkhorn, T=1000, M=4096, problem b: seed b,
            targets q.sample(4096, [b, 2])).  -> batch_cfg5_cases.npz
  tspio  -- the reference's tours (tsp.py:120-147) on config-5-like point sets
            and edge cases, and files its io.py wrote.  -> tsp_cases.npz, io/
  track  -- the reference's whole baseline_plan (tour + arc-length resampling +
            iterated TV-LQR tracking, tsp.py:150-316) for single_integrator_2d,
            diff_drive and aircraft_3d, and track_waypoints on a path with
            repeated points.  -> track_cases.npz
  large  -- shapes the reference cannot hold (it materialises C, C^T and
            C_xx): the oracle (oracle/flowcover_oracle.py, a streaming
            restatement checked bit-for-bit against the reference by
            tests/test_oracle_golden.py) computes cold and warm-started
            Sinkhorn flows at T=1e4 x M=1e5 (d=2) and T=2e4 x M=2e5 (d=3) on
            late-iteration-like states (X drawn from the target itself, so
            the flow is a small difference of barycentres -- the cancellation
            SURVEY hard part 2 warns about), three outer iterations of the
            config-3 planner (diff_drive, T=1e4, M=1e5), and fixed-h SVGD
            flows at T=2e4 (d=3).  Inputs are regenerated from seeds on the
            GPU box, so only outputs are stored.  -> large_cases.npz
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
WORKERS = os.cpu_count() or 1
os.environ.setdefault("FLOWCOVER_WORKERS", str(WORKERS))


def save(name: str, **arrays) -> None:
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


# ---------------------------------------------------------------------------
# inputs shared with tests/test_gpu_parity_r2.py (regenerated there)
# ---------------------------------------------------------------------------
LARGE = {
    # tag: (d, T, M)
    "L2": (2, 10_000, 100_000),
    "L3": (3, 20_000, 200_000),
}


def large_inputs(tag: str, mixture):
    """X: T draws of the target itself (seed stream [11, d]); Y: M draws, stream [0, 2]."""
    d, T, M = LARGE[tag]
    q = mixture(d)
    return q.sample(T, [11, d]), q.sample(M, [0, 2])


def step_along(X, a, size=2e-3):
    """The next planner-like state: X moved along the flow by `size` (max displacement)."""
    return X + size * a / np.abs(a).max()


# ---------------------------------------------------------------------------
def gen_plans():
    sys.path.insert(0, REF)
    import flowcover as fc
    from flowcover.seeding import STREAM_METRIC, STREAM_REFERENCE

    sys.path.insert(0, HERE)
    from make_golden import run_plan

    out = {}
    q2, q3 = fc.benchmark_mixture(2), fc.benchmark_mixture(3)
    cases = [
        ("dd_sk32", fc.differential_drive(), q2, "sinkhorn", 120.0, 20, 800),
        ("ac_sk32", fc.aircraft_3d(), q3, "sinkhorn", 120.0, 15, 800),
        ("ac_st32", fc.aircraft_3d(), q3, "stein", 0.1, 10, 1100),
    ]
    for tag, model, q, method, eta, iters, T in cases:
        tg = fc.SamplePoints(q.sample(2000, [0, STREAM_REFERENCE])) if method == "sinkhorn" else q
        cfg = fc.PlanConfig(method=method, eta=eta, max_iterations=iters, convergence_tol=0.0,
                            metric_interval=0, seed=0)
        res = run_plan(tag, model, tg, fc.Discretization(0.05, T, fc.default_start(model)), cfg,
                       record=True)
        draws = q.sample(2000, [0, STREAM_METRIC])
        res[f"{tag}_coverage"] = np.array(
            fc.coverage_metric(res[f"{tag}_S"], model, draws, fc.SinkhornConfig()))
        out.update(res)
    save("plan_fp32_cases.npz", **out)


def gen_batch():
    sys.path.insert(0, REF)
    import flowcover as fc
    from flowcover.seeding import STREAM_REFERENCE

    out = {}
    q = fc.benchmark_mixture(2)
    model = fc.single_integrator_2d()
    for b in range(3):
        tg = fc.SamplePoints(q.sample(4096, [b, STREAM_REFERENCE]))
        cfg = fc.PlanConfig(method="sinkhorn", eta=150.0, max_iterations=30, convergence_tol=0.0,
                            metric_interval=0, seed=b)
        t0 = time.perf_counter()
        res = fc.plan(model, tg, fc.Discretization(0.05, 1000, np.array([0.1, 0.1])), cfg)
        print(f"  cfg5 problem {b}: {time.perf_counter() - t0:.1f}s", flush=True)
        out[f"b{b}_S"] = res.trajectory.S
        out[f"b{b}_U"] = res.trajectory.U
        out[f"b{b}_flow_norms"] = res.flow_norms
        out[f"b{b}_lqr_costs"] = res.lqr_costs
    save("batch_cfg5_cases.npz", **out)


def gen_large(which: str = ""):
    sys.path.insert(0, ROOT)
    from oracle import flowcover_oracle as O

    out = {}
    for tag in LARGE:
        if which and tag not in which:
            continue
        X, Y = large_inputs(tag, O.benchmark_mixture)
        warm: dict = {}
        st1: dict = {}
        t0 = time.perf_counter()
        a1, c1, e1 = O.sinkhorn_flow(X, Y, "auto", 1000, 1e-6, warm, workers=WORKERS, stats=st1)
        f1, p1 = warm["f"].copy(), warm["p"].copy()
        X2 = step_along(X, a1)
        st2: dict = {}
        a2, c2, e2 = O.sinkhorn_flow(X2, Y, "auto", 1000, 1e-6, warm, workers=WORKERS, stats=st2)
        print(f"  {tag}: {time.perf_counter() - t0:.1f}s inner {st1} / {st2}", flush=True)
        out.update({
            f"{tag}_a1": a1, f"{tag}_f1": f1, f"{tag}_p1": p1,
            f"{tag}_a2": a2, f"{tag}_f2": warm["f"], f"{tag}_p2": warm["p"],
            f"{tag}_inner": np.array([st1["iters_cross"], st1["iters_self"],
                                      st2["iters_cross"], st2["iters_self"]]),
            f"{tag}_omega": np.array([st1["omega"], st2["omega"]]),
            f"{tag}_err": np.array([e1, e2]),
        })
    if not which or "S3" in which:
        # fixed-h SVGD flow at T=2e4, d=3 (config-4 SVGD with a fixed bandwidth)
        q3 = O.benchmark_mixture(3)
        Xs = q3.sample(20_000, [12, 3])
        t0 = time.perf_counter()
        a, _, _ = O.stein_flow(Xs, q3, 0.01, workers=WORKERS)
        print(f"  S3: {time.perf_counter() - t0:.1f}s", flush=True)
        out["S3_a"] = a
    if not which or "cfg3" in which:
        # config 3 (diff_drive, Sinkhorn, T=1e4, M=1e5, eta=1500): 3 outer iterations
        q2 = O.benchmark_mixture(2)
        Y = q2.sample(100_000, [0, 2])
        rec: list = []
        t0 = time.perf_counter()
        r = O.plan("diff_drive", np.array([0.1, 0.1, 0.0]), 0.05, 10_000, "sinkhorn", 1500.0, 3,
                   targets=Y, workers=WORKERS, record=rec)
        print(f"  cfg3: {time.perf_counter() - t0:.1f}s inner {r['inner']}", flush=True)
        out.update({"cfg3_S": r["S"], "cfg3_U": r["U"], "cfg3_flow_norms": r["flow_norms"],
                    "cfg3_lqr_costs": r["lqr_costs"], "cfg3_inner": np.array(r["inner"])})
        for i, (Si, ai) in enumerate(rec):
            out[f"cfg3_rec{i}_S"] = Si
            out[f"cfg3_rec{i}_a"] = ai
    name = "large_cases.npz" if not which else f"large_cases_{which.replace(',', '_')}.npz"
    save(name, **out)


def gen_tsp_io():
    """Reference tours (tsp.py:120-147) for config-5-like point sets and edge
    cases, and files written by the reference's io.py."""
    sys.path.insert(0, REF)
    import flowcover as fc
    from flowcover import io as rio
    from flowcover.tsp import build_tour

    out = {}
    q2, q3 = fc.benchmark_mixture(2), fc.benchmark_mixture(3)
    cases = [("t0", q2.sample(1000, [0, 2]), 0, None), ("t1", q2.sample(1000, [1, 2]), 1, None),
             ("t3d", q3.sample(300, [5, 2]), 5, None), ("tbud", q2.sample(400, [7, 2]), 7, 5),
             ("t2", np.array([[0.0, 0.0], [1.0, 1.0]]), 3, None),
             ("tdup", np.array([[0.5, 0.5]] * 4 + [[0.1, 0.2]] * 3), 2, None)]
    for tag, pts, seed, budget in cases:
        t0 = time.perf_counter()
        tour = build_tour(pts, seed, budget)
        print(f"  tour {tag}: {time.perf_counter() - t0:.1f}s length {tour.length:.6f}", flush=True)
        out.update({f"{tag}_pts": pts, f"{tag}_order": tour.order,
                    f"{tag}_meta": np.array([seed, -1 if budget is None else budget, tour.length])})
    save("tsp_cases.npz", **out)
    io_dir = os.path.join(HERE, "io")
    os.makedirs(io_dir, exist_ok=True)
    m = fc.differential_drive()
    U = 0.1 * np.random.default_rng(3).standard_normal((25, 2))
    S = fc.rollout(m, fc.default_start(m), U, 0.05)
    rio.write_trajectory(os.path.join(io_dir, "traj_diff_drive.csv"),
                         fc.Trajectory(S=S, U=U, dt=0.05), m)
    rio.write_points(os.path.join(io_dir, "points_named.csv"), q3.sample(17, [1, 9]),
                     names=("x", "y", "z"))
    rio.write_points(os.path.join(io_dir, "points_plain.csv"), q2.sample(9, [2, 9]))
    rio.write_metrics(os.path.join(io_dir, "metrics.json"),
                      {"coverage": 0.1234567890123, "iterations": 20, "method": "sinkhorn",
                       "phases": {"flow": 1.5, "lqr": 0.25}})
    print("  wrote io/*", flush=True)


def gen_track():
    """The reference's whole TSP baseline (tsp.py:276-316: targets, tour, arc-length
    resampling, iterated TV-LQR tracking) for the three liftable models, and
    track_waypoints on a path with repeated points (zero-length segments)."""
    sys.path.insert(0, REF)
    import flowcover as fc

    out = {}
    cases = [("si", fc.single_integrator_2d(), 2, 300, 0), ("dd", fc.differential_drive(), 2, 300, 1),
             ("ac", fc.aircraft_3d(), 3, 200, 2)]
    for tag, model, d, T, seed in cases:
        q = fc.benchmark_mixture(d)
        disc = fc.Discretization(0.05, T, fc.default_start(model))
        t0 = time.perf_counter()
        res = fc.baseline_plan(model, q, disc, fc.BaselineConfig(seed=seed))
        print(f"  baseline {tag}: {time.perf_counter() - t0:.1f}s", flush=True)
        out.update({f"{tag}_S": res.trajectory.S, f"{tag}_U": res.trajectory.U,
                    f"{tag}_order": res.tour.order, f"{tag}_waypoints": res.waypoints,
                    f"{tag}_meta": np.array([seed, T])})
    W = np.array([[0.1, 0.1], [0.1, 0.1], [0.4, 0.2], [0.4, 0.2], [0.4, 0.2], [0.7, 0.6],
                  [0.3, 0.8], [0.3, 0.8]])
    S, U = fc.track_waypoints(fc.differential_drive(), W, 120, 0.05, iterations=6)
    out.update({"rep_W": W, "rep_S": S, "rep_U": U})
    out["rs_in"] = W
    out["rs_out"] = fc.resample_arclength(W, 37)
    out["rs_single"] = fc.resample_arclength(W[:2], 5)
    save("track_cases.npz", **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="plans,batch,large,tspio,track")
    ap.add_argument("--large", default="", help="subset of L2,L3,S3,cfg3")
    args = ap.parse_args()
    jobs = dict(plans=gen_plans, batch=gen_batch, large=lambda: gen_large(args.large),
                tspio=gen_tsp_io, track=gen_track)
    for name, fn in jobs.items():
        if name not in args.only.split(","):
            continue
        t0 = time.perf_counter()
        fn()
        print(f"[{name}] {time.perf_counter() - t0:.1f}s", flush=True)
