"""Measure BASELINE.json configs beyond the bench workload (one GPU).

    python scripts/configs.py [cfg ...]      cfg in {1, 3, 4, 4s, 5, 5full}

5full: all 4096 config-5 problems in one batched launch on one GPU (the
8-GPU split runs 512 per rank through distributed.plan_batch).

Every config prints one JSON line: outer iterations timed, planner it/s,
executed pair evaluations per second over the whole planner step, and (for
Sinkhorn configs) a live replay of the asymmetric solve on the last iterate
with its fraction of the measured MUFU.EX2 peak.  Inputs follow SURVEY.md
§8(d): seed 0, benchmark_mixture draws from stream [0, 2], dt = 0.05.
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import _dev, _lib  # noqa: E402

import bench  # noqa: E402


def roofline_replay(X_last, Y, reps=5):
    """Time the chunked asymmetric solve (fp32, fixed 10 inner iterations) on the
    last iterate: the dominant kernel at configs 3-4 (point sets too large for
    the shared-memory resident path)."""
    from paper_2511_11514_b200 import _precision
    from paper_2511_11514_b200.sinkhorn import _resolve_on_device

    n, d = X_last.shape
    m = Y.shape[0]
    prec = _precision.pick("auto", n * max(n, m), 1e-6)
    dev = _dev.require_cuda()
    Xd, Yd = _dev.f64(X_last, dev), _dev.f64(Y, dev)
    scal = _resolve_on_device(_lib.FCB_OT_ASYM, prec, Xd, n, Yd, m, d, 0.0)
    lib = _lib.load()
    f, g, rs = _dev.empty((n,)), _dev.empty((m,)), _dev.empty((n,))
    stat, bary = _dev.empty((4,)), _dev.empty((n, d + 1))
    ws = _dev.Workspace.get(lib.fcb_ot_workspace_bytes(_lib.FCB_OT_ASYM, prec, n, m, d), "roof")
    iters = 10

    def launch():
        rc = lib.fcb_ot_solve(_lib.FCB_OT_ASYM, prec, _dev.ptr(Xd), n, _dev.ptr(Yd), m, d,
                              _dev.ptr(scal), iters, 1e-300, None, _dev.ptr(f), _dev.ptr(g),
                              _dev.ptr(rs), _dev.ptr(stat), _dev.ptr(bary), None, _dev.ptr(ws),
                              ws.numel(), _dev.stream())
        _lib.check(rc, "fcb_ot_solve")

    for _ in range(2):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    e1.synchronize()
    per_launch = e0.elapsed_time(e1) * 1e-3 / reps
    used = int(stat[1].item())
    pairs = 2.0 * used * n * m
    return {"pairs_per_launch": pairs, "seconds_per_launch": per_launch,
            "pairs_per_s": pairs / per_launch}


def timed_plan(model, q, disc, cfg, reps=1):
    fc.plan_detailed(model, q, disc, cfg)  # warm-up (allocations, module load)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    runs = []
    e0.record()
    for _ in range(reps):
        runs.append(fc.plan_detailed(model, q, disc, cfg))
    e1.record()
    e1.synchronize()
    return runs, e0.elapsed_time(e1) * 1e-3


def peak():
    return bench.measure_peak(torch, _lib.load())["ex2"]


def sinkhorn_cfg(name, model, T, M, iters, eta, d, solve_replay=True):
    q = fc.benchmark_mixture(d)
    Y = q.sample(M, [0, 2])
    disc = fc.Discretization(0.05, T, fc.default_start(model))
    cfg = fc.PlanConfig(method="sinkhorn", eta=eta, max_iterations=iters, convergence_tol=0.0,
                        metric_interval=0)
    runs, t = timed_plan(model, fc.SamplePoints(Y), disc, cfg)
    run = runs[-1]
    out = dict(config=name, T=T, M=M, outer_iterations=iters, seconds=t,
               planner_iters_per_s=iters / t, pairs=run.pairs, pairs_per_s=run.pairs / t,
               inner_iterations=[[int(a), int(b)] for a, b in run.flow_log[:, 1:3]],
               phase_s=dict(flow=run.result.phase_times.flow, lqr=run.result.phase_times.lqr,
                            rollout=run.result.phase_times.rollout))
    if solve_replay:
        X_last = model.project_states(run.result.trajectory.S[1:])
        rr = roofline_replay(X_last, Y, reps=3)
        pk = peak()
        out["solve_replay"] = dict(pairs_per_s=rr["pairs_per_s"], frac_of_mufu=rr["pairs_per_s"] / pk,
                                   mufu_peak=pk, ms_per_launch=rr["seconds_per_launch"] * 1e3,
                                   pairs_per_launch=rr["pairs_per_launch"])
    return out


def cfg1():
    di = fc.double_integrator_2d()
    q = fc.benchmark_mixture(2)
    disc = fc.Discretization(0.05, 500, np.array([0.1, 0.1, 0.0, 0.0]))
    cfg = fc.PlanConfig(method="stein", eta=0.1, max_iterations=100, convergence_tol=0.0,
                        metric_interval=0)
    runs, t = timed_plan(di, q, disc, cfg, reps=3)
    run = runs[-1]
    draws = q.sample(1000, [0, 3])
    cov = fc.coverage_metric(run.result.trajectory.S, di, draws)
    return dict(config="1: double integrator, SVGD median-h, T=500, 100 it", seconds=t / 3,
                planner_iters_per_s=100 * 3 / t, pairs_per_s=run.pairs * 3 / t, coverage=cov,
                phase_s=dict(flow=run.result.phase_times.flow, lqr=run.result.phase_times.lqr,
                             rollout=run.result.phase_times.rollout))


def cfg3():
    return sinkhorn_cfg("3: diff_drive, Sinkhorn, T=1e4, M=1e5", fc.differential_drive(), 10_000,
                        100_000, 5, 1500.0, 2)


def cfg4():
    return sinkhorn_cfg("4: aircraft_3d, Sinkhorn, T=1e5, M=1e6", fc.aircraft_3d(), 100_000,
                        1_000_000, 3, 15000.0, 3)


def cfg4s():
    """Config 4 SVGD part: Stein flow with a fixed bandwidth at T = 1e5 (d = 3)."""
    q = fc.benchmark_mixture(3)
    rng = np.random.default_rng(0)
    X = rng.random((100_000, 3))
    cfgS = fc.SteinConfig(bandwidth=0.01, precision="float32")
    fc.stein_flow(X, q, cfgS)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        fc.stein_flow(X, q, cfgS)
    t = (time.perf_counter() - t0) / reps
    pk = peak()
    return dict(config="4 (SVGD): Stein flow, fixed h, T=1e5, d=3 (incl. host copies)",
                seconds_per_flow=t, pairs_per_s=1e10 / t, frac_of_mufu=1e10 / t / pk)


def cfg5(problems=512, iters=100):
    """Config 5: independent T=1000, M=4096 single-integrator problems (problem b: seed b,
    targets from stream [b, 2]), 512 per GPU as in SURVEY 8(d), planned as ONE batched
    fused launch (one problem per CTA); a few problems through the per-problem loop
    for comparison."""
    m = fc.single_integrator_2d()
    q = fc.benchmark_mixture(2)
    probs = []
    for b in range(problems):
        Y = q.sample(4096, [b, 2])
        probs.append((m, fc.SamplePoints(Y), fc.Discretization(0.05, 1000, np.array([0.1, 0.1])),
                      fc.PlanConfig(method="sinkhorn", eta=150.0, max_iterations=iters,
                                    convergence_tol=0.0, metric_interval=0, seed=b)))
    fc.plan_batch_detailed(probs[:2])  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    runs = fc.plan_batch_detailed(probs)
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    pairs = sum(r.pairs for r in runs)
    pk = peak()
    # per-problem loop (one problem over the whole GPU at a time) on a sample
    os.environ["FCB_FUSED"] = "0"
    k = 4
    fc.plan_detailed(*probs[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    seq = [fc.plan_detailed(*p) for p in probs[:k]]
    torch.cuda.synchronize()
    t_seq = (time.perf_counter() - t0) / k
    os.environ["FCB_FUSED"] = "1"
    return dict(config=f"5: {problems} independent SI problems, T=1000, M=4096, {iters} it "
                       "(batched fused launch, one problem per CTA)",
                seconds=t, problems_per_s=problems / t, planner_iters_per_s=problems * iters / t,
                pairs=pairs, pairs_per_s=pairs / t, frac_of_mufu=pairs / t / pk, mufu_peak=pk,
                per_problem_loop_seconds_per_problem=t_seq,
                per_problem_loop_extrapolated_s=t_seq * problems,
                seq_pairs_per_s=sum(r.pairs for r in seq) / (t_seq * k))


if __name__ == "__main__":
    which = sys.argv[1:] or ["1", "3", "4", "4s", "5"]
    table = {"1": cfg1, "3": cfg3, "4": cfg4, "4s": cfg4s, "5": cfg5,
             "5full": lambda: cfg5(problems=4096)}
    for w in which:
        res = table[w]()
        print(json.dumps(res), flush=True)
