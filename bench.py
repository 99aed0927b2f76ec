#!/usr/bin/env python
"""Benchmark of the reference-flow generator (BASELINE.json metric).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
2D double integrator, Sinkhorn-divergence flow, T=2000 trajectory states,
M=10^4 reference samples (Gaussian-mixture draws, seed stream [0, 2]),
200 outer planner iterations, eta=300, dt=0.05, tol=1e-6, omega="auto".
One step = one complete plan() of that workload (rollout, flow, LQR and the
control update for 200 iterations).

metric  "flow-field pairwise evals/sec": executed (query, source) pair
        evaluations of the LSE sweeps (2 k_a T M + k_s T^2 per outer
        iteration, k_a / k_s the inner iteration counts the device actually
        ran) divided by the device-timed step time; planner iterations/s
        are reported alongside.
value   inputs resident in HBM (targets pre-staged), CUDA events on the
        launching stream over the K timed steps, max over ranks.
e2e     the public plan() with host numpy inputs (uploads + result
        download inside the timed region).
roofline  the dominant work: the Sinkhorn-flow phase of the persistent
        planner launch (rs_plan_kernel runs iterations 1..199 in one launch;
        iteration 0 runs rs_flow_kernel), timed live inside the timed region
        on the device (CUDA events around the iteration-0 flow launch,
        %globaltimer stamps around each in-kernel flow phase): executed
        pair-evals/s (= MUFU.EX2/s, one exp2 per pair) vs the MUFU.EX2 peak
        measured by the probe kernel in this run; traffic from the committed
        ncu capture.
cpu_baseline  the oracle port of the reference (numpy float64, row-chunked
        thread pool as in the reference) on this host's cores, on a bounded
        sample of the same workload (the first outer iterations).

--impl reference runs that CPU port as the reference arm.
--gpus N (torchrun): every rank runs its own independent problem (seed =
rank): independent planning problems split across ranks, weak scaling.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

T_STEPS = 2000
M_TARGETS = 10_000
ITERATIONS = 200
ETA = 300.0
DT = 0.05
S0 = np.array([0.1, 0.1, 0.0, 0.0])
METRIC = "flow-field pairwise evals/sec (T x M, executed LSE sweeps)"
UNIT = "pair-evals/s"
WORKLOAD = ("2D double integrator, Sinkhorn-divergence flow, T=2000, M=1e4, 200 iterations "
            "(BASELINE.json configs[1])")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def targets_for(seed: int) -> np.ndarray:
    from paper_2511_11514_b200.reference import benchmark_mixture

    return benchmark_mixture(2).sample(M_TARGETS, [seed, 2])


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
# our arm
# ---------------------------------------------------------------------------
def measure_peak(torch, lib, iters=4096):
    """MUFU.EX2 and FFMA throughput (ops/s) from the probe kernels."""
    from paper_2511_11514_b200 import _dev

    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    res = {}
    for which, name in ((0, "ex2"), (1, "ffma")):
        for _ in range(2):  # warm
            lib.fcb_peak_probe(which, iters, _dev.ptr(out), _dev.stream())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            lib.fcb_peak_probe(which, iters, _dev.ptr(out), _dev.stream())
        e1.record()
        e1.synchronize()
        ops = float(out[0].item()) * reps
        res[name] = ops / (e0.elapsed_time(e1) * 1e-3)
    return res


def load_traffic():
    """dram bytes per flow_kernel launch from the committed ncu --set full
    capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "flow_kernel_traffic.json")
    try:
        with open(path) as fh:
            rec = json.load(fh)
        return rec
    except (OSError, ValueError):
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    else:
        torch.cuda.set_device(0)
    import paper_2511_11514_b200 as fc
    from paper_2511_11514_b200 import _dev, _lib

    lib = _lib.load()
    model = fc.double_integrator_2d()
    Y = targets_for(rank)
    disc = fc.Discretization(DT, T_STEPS, S0)
    cfg = fc.PlanConfig(method="sinkhorn", eta=ETA, max_iterations=ITERATIONS,
                        convergence_tol=0.0, metric_interval=0, seed=rank)
    q = fc.SamplePoints(Y)
    Yd = _dev.f64(Y)
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

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- warm-up -------------------------------------------------------------
    for _ in range(args.warmup):
        fc.plan_detailed(model, q, disc, cfg, resident_targets=Yd)

    # ---- timed: inputs resident ---------------------------------------------
    runs = []
    barrier()
    launches0 = lib.fcb_launch_count()
    with ClockSampler(torch.cuda.current_device()) as clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            flush.zero_()  # 256 MiB > 126 MB L2 between steps
            runs.append(fc.plan_detailed(model, q, disc, cfg, resident_targets=Yd))
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        barrier()
    launches = lib.fcb_launch_count() - launches0
    t_dev = e0.elapsed_time(e1) * 1e-3
    pairs_local = sum(r.pairs for r in runs)
    t_max = max_over_ranks(t_dev)
    pairs_all = sum_over_ranks(pairs_local)
    iters_all = sum_over_ranks(float(sum(r.result.iterations_used for r in runs)))

    # ---- e2e: public API, host inputs -----------------------------------------
    barrier()
    h2d = Y.nbytes + T_STEPS * 2 * 8 + S0.nbytes
    d2h = 0
    e2e_pairs = 0.0
    ee0 = torch.cuda.Event(enable_timing=True)
    ee0.record()
    for _ in range(args.steps):
        flush.zero_()
        run = fc.plan_detailed(model, fc.SamplePoints(targets_for(rank)), disc, cfg)
        res = run.result
        d2h = (res.trajectory.S.nbytes + res.trajectory.U.nbytes + res.flow_norms.nbytes
               + res.lqr_costs.nbytes)
        e2e_pairs += run.pairs
    ee1 = torch.cuda.Event(enable_timing=True)
    ee1.record()
    barrier()
    t_e2e = max_over_ranks(ee0.elapsed_time(ee1) * 1e-3)
    e2e_pairs_all = sum_over_ranks(e2e_pairs)

    # ---- roofline of the dominant kernel (live, inside the timed region) -----
    # plan() runs iteration 0 as separate launches (rollout, rs_flow_kernel,
    # Riccati + update) and iterations 1.. as ONE persistent rs_plan_kernel
    # launch; the flow phase time of every iteration is device time (CUDA
    # events around the iteration-0 flow launch, %globaltimer stamps of the
    # flow phase inside rs_plan_kernel).  Algorithmic work: one exp2 per
    # (query, source) pair of every executed LSE sweep.
    roof = None
    if rank == 0:
        peak = measure_peak(torch, lib)
        ex2_peak = peak["ex2"]
        t_flow = sum(r.result.phase_times.flow for r in runs)
        t_total = sum(r.result.phase_times.total for r in runs)
        n_launch = sum(r.result.iterations_used for r in runs)
        achieved = pairs_local / max(t_flow, 1e-12)
        tr = load_traffic()
        roof = {
            "bound": "mufu",
            "kernel": "rs_plan_kernel<2,1,DoubleIntegrator> flow phase (shared-memory-resident "
                      "Sinkhorn flow: omega, packs, asymmetric + self solves, envelope gradient)",
            "achieved": achieved / 1e9,
            "peak": ex2_peak / 1e9,
            "unit": "Gexp/s",
            "frac": achieved / ex2_peak,
            "traffic": (tr["dram_bytes_per_launch"] if tr else None),
            "traffic_source": (tr["source"] if tr else None),
            "algorithmic_bytes_per_launch": (tr["algorithmic_bytes_per_launch"] if tr else None),
            "peak_source": "measured MUFU.EX2 probe (fcb_peak_probe) in this run",
            "ffma_peak_Gops": peak["ffma"] / 1e9,
            "algorithmic": "1 exp2 per pair; pairs/launch = 2*k_a*T*M + k_s*T^2 (executed)",
            "launches": n_launch,
            "pairs_per_launch": pairs_local / max(n_launch, 1),
            "ms_per_launch": t_flow / max(n_launch, 1) * 1e3,
            "share_of_step": t_flow / max(t_total, 1e-12),
        }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_iterations)

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": METRIC,
            "value": pairs_all / t_max,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "fp32 pairwise sweeps (MUFU ex2), fp64 potentials/LQR/rollout",
            "data": "synthetic: benchmark_mixture(2) draws, seed stream [rank, 2]",
            "config": {
                "workload": WORKLOAD,
                "T": T_STEPS, "M": M_TARGETS, "outer_iterations": ITERATIONS, "eta": ETA,
                "problems": world, "parallelism": f"independent problems x{world}",
                "l2": "256 MiB memset between steps (inputs < L2)",
            },
            "planner_iters_per_s": iters_all / t_max,
            "pairs_per_step": pairs_all / args.steps / world,
            "e2e": {"value": e2e_pairs_all / t_e2e, "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": t_e2e / args.steps * 1e3},
            "gpu_launches": int(launches),
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU (reference port) arm
# ---------------------------------------------------------------------------
def cpu_sample(outer: int, workers: int, seed: int = 0) -> tuple[float, float, float]:
    """First `outer` iterations of the workload on the oracle port; (seconds, pairs, iters)."""
    from oracle import flowcover_oracle as O

    Y = targets_for(seed)
    t0 = time.perf_counter()
    r = O.plan("double_integrator_2d", S0, DT, T_STEPS, "sinkhorn", ETA, outer, targets=Y,
               seed=seed, workers=workers)
    dt = time.perf_counter() - t0
    pairs = sum(2.0 * ka * T_STEPS * M_TARGETS + ks * T_STEPS * T_STEPS for ka, ks in r["inner"])
    return dt, pairs, float(len(r["flow_norms"]))


def cpu_baseline(outer: int) -> dict:
    workers = os.cpu_count() or 1
    dt, pairs, iters = cpu_sample(outer, workers)
    return {"value": pairs / dt, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"first {outer} outer iterations of the workload (numpy float64 oracle, "
                      f"{workers} threads)", "seconds": dt,
            "planner_iters_per_s": iters / dt}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    outer = args.ref_outer
    for _ in range(args.warmup):
        cpu_sample(1, workers)
    tot_t = tot_p = tot_i = 0.0
    for _ in range(args.steps):
        dt, pairs, iters = cpu_sample(outer, workers)
        tot_t += dt
        tot_p += pairs
        tot_i += iters
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
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: benchmark_mixture(2) draws, seed stream [0, 2]",
        "config": {"workload": WORKLOAD, "T": T_STEPS, "M": M_TARGETS,
                   "sample_per_step": f"{outer} outer iterations"},
        "planner_iters_per_s": tot_i / tot_t,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": f"{outer} outer iterations per step, oracle port of the "
                                   f"reference (numpy float64, {workers} threads)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-iterations", type=int, default=6)
    ap.add_argument("--ref-outer", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
