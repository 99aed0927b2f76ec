#!/usr/bin/env python
"""Benchmark of the reference-flow generator (BASELINE.json metric).

Headline workload: BASELINE.json configs[3] -- the north_star's target shape.
  aircraft_3d (the reference's 3D model, standing in for "quadrotor-style"),
  T = 1e5 trajectory states, M = 1e6 reference samples (benchmark_mixture(3)
  draws, seed stream [0, 2]), dt = 0.05, SVGD + Sinkhorn.
  One step = 3 outer planner iterations with the Sinkhorn-divergence flow
  (eta 15000 = 0.15 T, omega "auto", tol 1e-6, cold start) followed by 3 with
  the SVGD flow (fixed h = 0.01, eta 0.1): rollout, flow, LQR and the control
  update of every iteration, i.e. two complete plan() calls.
  --gpus N (N > 1): the reference samples / SVGD sources are sharded over the
  N ranks (distributed.py: M-sharded Sinkhorn, source-sharded SVGD) and the
  total work is fixed -- strong scaling.  Without torchrun, bench.py launches
  its own N ranks.

metric  "flow-field pairwise evals/sec": executed (query, source) pair
        evaluations -- Sinkhorn 2 k_a T M + k_s T^2 per outer iteration (k_a,
        k_s the inner iterations the device ran), SVGD T^2 -- divided by the
        device-timed step time (max over ranks); planner iterations/s alongside.
value   inputs resident in HBM; CUDA events on the launching stream; a 256 MiB
        memset between steps flushes the 126 MB L2 (inputs are smaller).
e2e     the public plan() with host numpy inputs (target upload and result
        download inside the timed region).
roofline  the flow phases (Sinkhorn flow_kernel, SVGD kernels), device-timed
        inside the timed region (CUDA events around every flow launch), against
        the hardware roof of the executed instruction mix: one MUFU.EX2 per
        pair, and FP32 lane-ops per pair of d+2 (LSE sweeps), 2d+2
        (barycentre/self sweeps) and 3d+1 (SVGD); MUFU.EX2 and FFMA peaks
        measured live by the probe kernel.  frac = (time at the roof) /
        (measured flow time); frac_of_mufu and the SURVEY.md 8(d) composite
        (2d+2 / 3d+2 ops per pair) alongside.
cpu_baseline  the oracle port of the reference (numpy float64, all host
        threads) on a bounded sample of the same workload; the full step is
        infeasible on CPU (the reference would materialise 2 TB of cost
        matrices), so the step time is extrapolated from the sample's rate.
secondary  N=1 only, device-timed like `value`: configs[1] (2D double
        integrator, Sinkhorn, T=2000, M=1e4, 200 iterations; the round-1
        headline), configs[0] (SVGD median h, T=500, 100 iterations:
        planner it/s), configs[2] (diff_drive, T=1e4, M=1e5) and configs[4]
        (512 independent problems per GPU in one batched launch).

--impl reference runs the oracle port's sample as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ---- config 4 (headline) ---------------------------------------------------------
T4, M4, D4 = 100_000, 1_000_000, 3
SK_ITERS, SV_ITERS = 3, 3
ETA_SK, ETA_SV, H_SV = 15_000.0, 0.1, 0.01
DT = 0.05
METRIC = "flow-field pairwise evals/sec (T x M, executed LSE / SVGD sweeps)"
UNIT = "pair-evals/s"
WORKLOAD = ("BASELINE configs[3]: aircraft_3d (3D quadrotor-style), T=1e5, M=1e6, "
            "SVGD + Sinkhorn; step = 3 Sinkhorn-flow + 3 SVGD (fixed h) planner iterations")
# ---- config 2 (secondary) -----------------------------------------------------------
T2, M2, IT2, ETA2 = 2000, 10_000, 200, 300.0
S0_DI = np.array([0.1, 0.1, 0.0, 0.0])
# ---- CPU sample ----------------------------------------------------------------------
CPU_ROWS, CPU_SV = 400, 8000


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


_TARGETS = []


def targets4():
    if not _TARGETS:
        from paper_2511_11514_b200.reference import benchmark_mixture

        _TARGETS.append(benchmark_mixture(D4).sample(M4, [0, 2]))
    return _TARGETS[0]


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------
def measure_peak(torch, lib, iters=4096):
    """MUFU.EX2 and FFMA throughput (ops/s) from the probe kernels."""
    from paper_2511_11514_b200 import _dev

    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    res = {}
    for which, name in ((0, "ex2"), (1, "ffma")):
        for _ in range(2):
            lib.fcb_peak_probe(which, iters, _dev.ptr(out), _dev.stream())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            lib.fcb_peak_probe(which, iters, _dev.ptr(out), _dev.stream())
        e1.record()
        e1.synchronize()
        res[name] = float(out[0].item()) * reps / (e0.elapsed_time(e1) * 1e-3)
    return res


def load_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def sweep_pairs(run, T, M):
    """(LSE-only pairs, barycentre-sweep pairs) of a Sinkhorn plan run."""
    ka, ks = run.flow_log[:, 1], run.flow_log[:, 2]
    return float((ka * T * M).sum()), float((ka * T * M + ks * T * T).sum())


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
        group = dist.group.WORLD
    else:
        torch.cuda.set_device(0)
        group = None
    import paper_2511_11514_b200 as fc
    from paper_2511_11514_b200 import _dev, _lib
    from paper_2511_11514_b200.distributed import shard_rows

    lib = _lib.load()
    model = fc.aircraft_3d()
    Y = targets4()
    Y_mine = shard_rows(Y, rank, world) if world > 1 else Y
    q3 = fc.benchmark_mixture(D4)
    disc = fc.Discretization(DT, T4, fc.default_start(model))
    cfg_sk = fc.PlanConfig(method="sinkhorn", eta=ETA_SK, max_iterations=SK_ITERS,
                           convergence_tol=0.0, metric_interval=0, seed=0)
    cfg_sv = fc.PlanConfig(method="stein", eta=ETA_SV, max_iterations=SV_ITERS,
                           convergence_tol=0.0, metric_interval=0, seed=0,
                           stein=fc.SteinConfig(bandwidth=H_SV))
    Yd = _dev.f64(Y_mine)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step(resident: bool):
        if resident:
            sk = fc.plan_detailed(model, fc.SamplePoints(Y), disc, cfg_sk, resident_targets=Yd,
                                  group=group)
        else:
            sk = fc.plan_detailed(model, fc.SamplePoints(Y), disc, cfg_sk, group=group)
        sv = fc.plan_detailed(model, q3, disc, cfg_sv, group=group)
        return sk, sv

    for _ in range(args.warmup):
        step(True)

    # ---- timed: inputs resident -------------------------------------------------
    runs = []
    barrier()
    launches0 = lib.fcb_launch_count()
    with ClockSampler(torch.cuda.current_device()) as clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            flush.zero_()
            runs.append(step(True))
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        barrier()
    launches = lib.fcb_launch_count() - launches0
    t_max = max_over_ranks(e0.elapsed_time(e1) * 1e-3)
    pairs = sum(sk.pairs + sv.pairs for sk, sv in runs)  # whole-job pairs (same on all ranks)
    iters = sum(sk.result.iterations_used + sv.result.iterations_used for sk, sv in runs)

    # ---- e2e: public plan() with host inputs ------------------------------------------
    barrier()
    h2d = d2h = 0
    e2e_pairs = 0.0
    ee0 = torch.cuda.Event(enable_timing=True)
    ee0.record()
    for _ in range(args.steps):
        flush.zero_()
        sk, sv = step(False)
        h2d = Y_mine.nbytes + 2 * (T4 * 3 * 8 + 6 * 8)  # targets, initial controls, s0
        d2h = sum(r.result.trajectory.S.nbytes + r.result.trajectory.U.nbytes
                  + r.result.flow_norms.nbytes + r.result.lqr_costs.nbytes for r in (sk, sv))
        e2e_pairs += sk.pairs + sv.pairs
    ee1 = torch.cuda.Event(enable_timing=True)
    ee1.record()
    barrier()
    t_e2e = max_over_ranks(ee0.elapsed_time(ee1) * 1e-3)

    # ---- roofline of the flow phases ------------------------------------------------
    peak = measure_peak(torch, lib)
    lse, bary = 0.0, 0.0
    for sk, _ in runs:
        a, b = sweep_pairs(sk, T4, M4)
        lse += a
        bary += b
    svp = sum(sv.pairs for _, sv in runs)
    # hardware roof of the instruction mix the kernels execute: 1 MUFU.EX2 per
    # pair everywhere; FP32 lane-ops per pair: LSE sweep d+2 (w + rc, d FMAs,
    # the sum), barycentre sweep 2d+2 (+ d moment FMAs), SVGD 3d+1 (direct
    # form: d subtractions, d FMAs, the sum, d moment FMAs)
    hw = {"lse": min(peak["ex2"], peak["ffma"] / (D4 + 2)),
          "bary": min(peak["ex2"], peak["ffma"] / (2 * D4 + 2)),
          "svgd": min(peak["ex2"], peak["ffma"] / (3 * D4 + 1))}
    t_roof = lse / hw["lse"] + bary / hw["bary"] + svp / hw["svgd"]
    # SURVEY.md 8(d)'s algorithmic counts (2d+2 LSE, 3d+2 barycentre / SVGD)
    sv_lse = min(peak["ex2"], peak["ffma"] / (2 * D4 + 2))
    sv_bary = min(peak["ex2"], peak["ffma"] / (3 * D4 + 2))
    t_roof_survey = lse / sv_lse + (bary + svp) / sv_bary
    t_flow_local = sum(sk.result.phase_times.flow + sv.result.phase_times.flow for sk, sv in runs)
    t_flow = max_over_ranks(t_flow_local)
    t_flow_sk = sum(sk.result.phase_times.flow for sk, _ in runs)
    t_total = sum(sk.result.phase_times.total + sv.result.phase_times.total for sk, sv in runs)
    tr = load_json("r02/flow_kernel_traffic_cfg4.json")
    fpairs = lse + bary + svp
    roof = {
        "bound": "mufu (1 ex2 per pair); fp32 co-limits the barycentre sweeps (8 FP32 "
                 "lane-ops per pair at d=3) and SVGD (10): composite of per-sweep roofs",
        "kernel": ("flow_kernel<float,3,3> (chunked fp32 Sinkhorn flow, cross + self solves) + "
                   "sv_sweep_f32_kernel<3,4> (packed SVGD)" if world == 1 else
                   "sharded lse sweeps (ot_solve_kernel SWEEP mode) + sv_sweep_f32_kernel"),
        "achieved": fpairs / t_flow / 1e9,
        "peak": fpairs / t_roof / 1e9,
        "unit": "Gpair/s",
        "frac": t_roof / t_flow,
        "traffic": (tr["dram_bytes_per_launch"] if tr else None),
        "traffic_source": (tr["source"] if tr else None),
        "algorithmic_bytes_per_launch": (tr["algorithmic_bytes_per_launch"] if tr else None),
        "pairs": {"lse_only": lse, "barycentre_and_self": bary, "svgd": svp},
        "roofs_Gpair_s": {k: v / 1e9 for k, v in hw.items()},
        "frac_of_mufu": fpairs / t_flow / peak["ex2"],
        "survey_composite": {"peak": fpairs / t_roof_survey / 1e9,
                             "frac": t_roof_survey / t_flow,
                             "note": "SURVEY 8(d) charges 2d+2 / 3d+2 FP32 ops per pair; the "
                                     "expanded form executes d+2 / 2d+2, so this frac can exceed "
                                     "the hardware one"},
        "peaks_measured": {"mufu_ex2_Gops": peak["ex2"] / 1e9, "ffma_Gops": peak["ffma"] / 1e9,
                           "source": "fcb_peak_probe in this run"},
        "sinkhorn_flow_Gpair_s": (lse + bary) / max(t_flow_sk, 1e-12) / 1e9,
        "sinkhorn_flow_frac_of_mufu": (lse + bary) / max(t_flow_sk, 1e-12) / peak["ex2"],
        "ms_flow_per_step": t_flow / args.steps * 1e3,
        "share_of_step": t_flow_local / max(t_total, 1e-12),
        "launches_flow": int(sum(sk.result.iterations_used + sv.result.iterations_used
                                 for sk, sv in runs)),
    }

    cpu = None
    secondary = None
    if rank == 0 and world == 1:
        if not args.no_secondary:
            secondary = {
                "configs[1]": config2_secondary(torch, fc, _dev, lib, peak, min(args.steps, 10),
                                                flush),
                "configs[0]": config1_secondary(torch, fc, flush),
                "configs[2]": config3_secondary(torch, fc, _dev, peak, flush),
                "configs[4]": config5_secondary(torch, fc, peak),
                "configs[4].tsp_baseline": tsp_baseline_secondary(torch, fc),
            }
        if not args.no_cpu:
            sk0 = runs[0][0]
            cpu = cpu_baseline(sk0, pairs / args.steps)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": pairs / t_max,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "fp32 pairwise sweeps (MUFU ex2), fp64 potentials/LQR/rollout",
            "data": "synthetic: benchmark_mixture(3) draws (seed stream [0, 2]), "
                    "random-small initial controls (stream [0, 1])",
            "config": {
                "workload": WORKLOAD, "T": T4, "M": M4, "d": D4,
                "sinkhorn_iterations": SK_ITERS, "svgd_iterations": SV_ITERS,
                "eta_sinkhorn": ETA_SK, "eta_svgd": ETA_SV, "svgd_bandwidth": H_SV,
                "parallelism": ("single GPU" if world == 1 else
                                f"M-sharded Sinkhorn + source-sharded SVGD over {world} GPUs"),
                "l2": "256 MiB memset between steps (inputs < L2)",
            },
            "planner_iters_per_s": iters / t_max,
            "pairs_per_step": pairs / args.steps,
            "e2e": {"value": e2e_pairs / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": t_e2e / args.steps * 1e3},
            "gpu_launches": int(launches),
            "roofline": roof,
            "cpu_baseline": cpu,
            "secondary": secondary,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def config2_secondary(torch, fc, _dev, lib, peak, steps, flush):
    """BASELINE configs[1] on one GPU: the round-1 headline, for continuity."""
    model = fc.double_integrator_2d()
    Y = fc.benchmark_mixture(2).sample(M2, [0, 2])
    disc = fc.Discretization(DT, T2, S0_DI)
    cfg = fc.PlanConfig(method="sinkhorn", eta=ETA2, max_iterations=IT2, convergence_tol=0.0,
                        metric_interval=0, seed=0)
    q = fc.SamplePoints(Y)
    Yd = _dev.f64(Y)
    for _ in range(3):
        fc.plan_detailed(model, q, disc, cfg, resident_targets=Yd)
    torch.cuda.synchronize()
    runs = []
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        flush.zero_()
        runs.append(fc.plan_detailed(model, q, disc, cfg, resident_targets=Yd))
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    pairs = sum(r.pairs for r in runs)
    t_flow = sum(r.result.phase_times.flow for r in runs)
    return {"workload": "BASELINE configs[1]: 2D double integrator, Sinkhorn, T=2000, M=1e4, "
                        "200 iterations (persistent rs_plan_kernel)",
            "value": pairs / t, "unit": UNIT, "steps": steps, "ms_per_step": t / steps * 1e3,
            "planner_iters_per_s": sum(r.result.iterations_used for r in runs) / t,
            "flow_phase_frac_of_mufu": pairs / t_flow / peak["ex2"],
            "flow_share_of_step": t_flow / t}


def _timed(torch, fn, reps, flush=None):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    e0.record()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        out.append(fn())
    e1.record()
    e1.synchronize()
    return out, e0.elapsed_time(e1) * 1e-3


def config1_secondary(torch, fc, flush):
    """BASELINE configs[0]: 2D double integrator, SVGD with the exact median
    bandwidth, T=500, 100 iterations (the CPU-oracle config; iterations/s)."""
    di = fc.double_integrator_2d()
    q = fc.benchmark_mixture(2)
    disc = fc.Discretization(DT, 500, S0_DI)
    cfg = fc.PlanConfig(method="stein", eta=0.1, max_iterations=100, convergence_tol=0.0,
                        metric_interval=0, seed=0)
    runs, t = _timed(torch, lambda: fc.plan_detailed(di, q, disc, cfg), 5, flush)
    its = sum(r.result.iterations_used for r in runs)
    return {"workload": "BASELINE configs[0]: 2D double integrator, SVGD (median h), T=500, "
                        "100 iterations", "planner_iters_per_s": its / t,
            "ms_per_plan": t / len(runs) * 1e3, "pair_evals_per_s": sum(r.pairs for r in runs) / t}


def config3_secondary(torch, fc, _dev, peak, flush):
    """BASELINE configs[2]: diff_drive, Sinkhorn, T=1e4, M=1e5 (3 outer iterations)."""
    m = fc.differential_drive()
    Y = fc.benchmark_mixture(2).sample(100_000, [0, 2])
    Yd = _dev.f64(Y)
    disc = fc.Discretization(DT, 10_000, fc.default_start(m))
    cfg = fc.PlanConfig(method="sinkhorn", eta=1500.0, max_iterations=3, convergence_tol=0.0,
                        metric_interval=0, seed=0)
    runs, t = _timed(torch, lambda: fc.plan_detailed(m, fc.SamplePoints(Y), disc, cfg,
                                                      resident_targets=Yd), 3, flush)
    pairs = sum(r.pairs for r in runs)
    t_flow = sum(r.result.phase_times.flow for r in runs)
    return {"workload": "BASELINE configs[2]: diff_drive, Sinkhorn, T=1e4, M=1e5, 3 outer iterations",
            "value": pairs / t, "unit": UNIT, "ms_per_plan": t / len(runs) * 1e3,
            "flow_frac_of_mufu": pairs / t_flow / peak["ex2"]}


def config5_secondary(torch, fc, peak, problems=512, iters=100):
    """BASELINE configs[4] per GPU: 512 independent single-integrator problems
    (T=1000, M=4096; problem b: seed b, targets q.sample(4096, [b, 2])) in one
    batched launch, 100 iterations each."""
    m = fc.single_integrator_2d()
    q = fc.benchmark_mixture(2)
    probs = [(m, fc.SamplePoints(q.sample(4096, [b, 2])),
              fc.Discretization(DT, 1000, np.array([0.1, 0.1])),
              fc.PlanConfig(method="sinkhorn", eta=150.0, max_iterations=iters,
                            convergence_tol=0.0, metric_interval=0, seed=b))
             for b in range(problems)]
    runs, t = _timed(torch, lambda: fc.plan_batch_detailed(probs), 1)
    runs = runs[0]
    pairs = sum(r.pairs for r in runs)
    return {"workload": f"BASELINE configs[4] per GPU: {problems} independent problems, T=1000, "
                        f"M=4096, {iters} iterations, one batched launch",
            "seconds": t, "problems_per_s": problems / t, "value": pairs / t, "unit": UNIT,
            "frac_of_mufu": pairs / t / peak["ex2"]}


def tsp_baseline_secondary(torch, fc, problems=512):
    """BASELINE configs[4]'s comparison method, the TSP-waypoint baseline
    (tsp.py:276-316), on the GPU: every tour in one launch, then the tracking
    rounds per problem (baseline_plans); beside it the reference's own
    baseline_plan measured on the B200 box's host cores."""
    m = fc.single_integrator_2d()
    q = fc.benchmark_mixture(2)
    disc = fc.Discretization(DT, 1000, np.array([0.1, 0.1]))
    cfgs = [fc.BaselineConfig(seed=b) for b in range(problems)]
    _, t = _timed(torch, lambda: fc.baseline_plans(m, q, disc, cfgs), 1)
    ref = load_json("r02/tsp_baseline_cfg5_gpubox.json") or {}
    return {"workload": f"TSP-waypoint baseline, {problems} config-5 problems (tour + 10 TV-LQR "
                        "tracking rounds each), batched tours",
            "seconds": t, "seconds_per_problem": t / problems,
            "reference_host": {k: ref.get(k) for k in (
                "what", "host_cores", "processes", "mean_seconds_per_problem",
                "problems_per_second_all_processes", "extrapolated_4096_problems_seconds")}}


# ---------------------------------------------------------------------------
# CPU (reference port): a bounded sample of the config-4 step
# ---------------------------------------------------------------------------
def cpu_sample(workers: int, X0=None):
    """One inner Sinkhorn iteration (g-sweep of all M samples over CPU_ROWS
    trajectory points, f-sweep of those rows over all M) and one fixed-h SVGD
    flow on CPU_SV points, on the oracle port.  Returns (seconds, pairs)."""
    from oracle import flowcover_oracle as O

    Y = targets4()
    q = O.benchmark_mixture(D4)
    if X0 is None:
        X0 = q.sample(CPU_ROWS, [5, 3])
    X = X0[:CPU_ROWS]
    Xs = q.sample(CPU_SV, [6, 3])
    w = O.resolve_omega("auto", X, Y)
    f = np.zeros(X.shape[0])
    t0 = time.perf_counter()
    Lg = O.lse_sweep(Y, X, f, w, workers=workers)
    g = w * (-np.log(Y.shape[0]) - Lg)
    O.lse_sweep(X, Y, g, w, workers=workers)
    O.stein_flow(Xs, q, H_SV, workers=workers)
    dt = time.perf_counter() - t0
    return dt, 2.0 * X.shape[0] * Y.shape[0] + float(CPU_SV) ** 2


def cpu_baseline(sk_run, pairs_per_step) -> dict:
    workers = os.cpu_count() or 1
    X0 = sk_run.result.trajectory.S[1:, :3]
    cpu_sample(workers, X0)  # warm (imports, page-in)
    dt, pairs = cpu_sample(workers, X0)
    rate = pairs / dt
    return {"value": rate, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": (f"one inner Sinkhorn iteration of {CPU_ROWS} trajectory rows x M=1e6 "
                       f"(g- and f-sweep) + one SVGD flow on {CPU_SV} points, numpy float64 "
                       f"oracle, {workers} threads"),
            "seconds": dt,
            "extrapolated_seconds_per_step": pairs_per_step / rate,
            "extrapolated": True}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(workers)
    tot_t = tot_p = 0.0
    for _ in range(args.steps):
        dt, pairs = cpu_sample(workers)
        tot_t += dt
        tot_p += pairs
    v = tot_p / tot_t
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": tot_t / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: benchmark_mixture(3) draws (seed stream [0, 2])",
        "config": {"workload": WORKLOAD, "T": T4, "M": M4, "d": D4,
                   "sample_per_step": (f"one inner Sinkhorn iteration on {CPU_ROWS} rows x "
                                       f"M=1e6 + one SVGD flow on {CPU_SV} points")},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": "as config.sample_per_step; numpy float64 oracle port of "
                                   f"the reference, {workers} threads"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args) -> int:
    """--gpus N without torchrun: start N ranks (one per GPU) and relay rank 0."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    _, world, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
