"""The sharded flows' device steps (csrc/shard.cu) on one GPU.

The collective schedule at world sizes > 1 is covered on CPU by
test_distributed_gloo (CPU stand-in of these steps, tests/shard_cpu_ops.py).
Here the CUDA steps are checked (a) end to end at world size 1 against the
oracle and the single-GPU flows, (b) step by step against the CPU stand-in on
synthetic gathered buffers of R = 3 shards -- the merge paths a multi-GPU run
takes -- and (c) through plan_detailed(group=...) against the reference's
golden plans.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2511_11514_b200 as fc
from fcb_testutil import load_golden, rel_inf
from oracle import flowcover_oracle as O
from paper_2511_11514_b200 import _lib
from paper_2511_11514_b200 import distributed as D
from paper_2511_11514_b200.seeding import STREAM_REFERENCE
from shard_cpu_ops import CpuOps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group1():
    """A one-rank NCCL process group (the sharded code path at world size 1)."""
    if dist.is_initialized():
        yield dist.group.WORLD
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("n,m,d,precision", [(300, 500, 2, "float64"), (2000, 10_000, 2, "auto"),
                                             (1500, 6000, 3, "auto")])
def test_sharded_flow_world1_matches_oracle(n, m, d, precision):
    q = O.benchmark_mixture(d)
    X, Y = q.sample(n, [31, d]), q.sample(m, [0, 2])
    cfg = fc.SinkhornConfig(precision=precision)
    flow = D.ShardedSinkhornFlow(Y, cfg)
    st1, st2 = {}, {}
    a1 = flow(X, stats=st1).a
    X2 = X + 1e-3
    a2 = flow(X2, stats=st2).a
    warm: dict = {}
    s1, s2 = {}, {}
    ref1, _, _ = O.sinkhorn_flow(X, Y, warm=warm, workers=os.cpu_count() or 1, stats=s1)
    ref2, _, _ = O.sinkhorn_flow(X2, Y, warm=warm, workers=os.cpu_count() or 1, stats=s2)
    assert (st1["iters_cross"], st1["iters_self"]) == (s1["iters_cross"], s1["iters_self"])
    assert (st2["iters_cross"], st2["iters_self"]) == (s2["iters_cross"], s2["iters_self"])
    tol = 1e-9 if precision == "float64" else 1e-4
    assert rel_inf(a1, ref1) <= tol, rel_inf(a1, ref1)
    assert rel_inf(a2, ref2) <= tol, rel_inf(a2, ref2)


def _rand_gather(rng, R, n, d):
    g = np.empty((R, n, d + 1))
    g[:, :, 0] = rng.normal(scale=3.0, size=(R, n)) - 5.0
    g[:, :, 1:] = rng.random((R, n, d))
    return g


@pytest.mark.parametrize("d", [1, 2, 3])
def test_cross_merge_and_self_commit_kernels_R3(d):
    """The R > 1 merge paths of the CUDA steps vs the CPU stand-in."""
    rng = np.random.default_rng(d)
    n, R = 1001, 3
    dev, cpu = D.DeviceOps(), CpuOps()
    gath = _rand_gather(rng, R, n, d)
    f0 = rng.normal(scale=0.01, size=n)
    chunk = (n + R - 1) // R
    gs = np.zeros((R, chunk, d + 4))
    for r in range(R):
        lo, hi = D.shard_bounds(n, r, R)
        gs[r, : hi - lo] = rng.random((hi - lo, d + 4))
    out = {}
    for name, ops in (("gpu", dev), ("cpu", cpu)):
        t = ops.tensor
        scal = t(np.r_[0.03, np.zeros(15)])
        f, fnext = t(f0), ops.zeros((n,))
        rs, mass, ybar = ops.zeros((n,)), ops.zeros((n,)), ops.zeros((n, d))
        ctl = ops.zeros((8,), dtype=torch.int32)
        eslot = ops.zeros((2,), dtype=torch.int64)
        stat = ops.zeros((4,))
        ops.cross_merge(n, d, R, t(gath), scal, 1e-6, 5, f, fnext, rs, mass, ybar, ctl, eslot, stat)
        p, pnext = t(f0), ops.zeros((n,))
        rho, massp, xbar = ops.zeros((n,)), ops.zeros((n,)), ops.zeros((n, d))
        stat_p = ops.zeros((4,))
        ops.self_commit(n, d, R, chunk, t(gs), 1e-6, 1, p, pnext, rho, massp, xbar, ctl, eslot,
                        stat_p)
        out[name] = [x.cpu().numpy() for x in (f, fnext, rs, mass, ybar, stat, ctl, p, rho, xbar,
                                               stat_p)]
    for a, b in zip(out["gpu"], out["cpu"]):
        np.testing.assert_allclose(a, b, rtol=1e-13, atol=0)


@pytest.mark.parametrize("d", [2, 3])
def test_stein_partial_and_combine_kernels_R3(d):
    """Source-sharded SVGD: three column ranges summed in rank order equal the
    single-GPU flow (and the oracle)."""
    q = O.benchmark_mixture(d)
    X = q.sample(2500, [41, d])
    n, R = X.shape[0], 3
    dev = D.DeviceOps()
    Xd = dev.tensor(X)
    fq = fc.benchmark_mixture(d)
    k, params = dev.mixture_params(fq)
    scores = dev.zeros((n, d))
    dev.gmm_score(Xd, k, params, scores, None)
    hstat = dev.tensor([0.02, np.nan, 0.0, 0.0])
    parts = dev.zeros((R, n, d + 1))
    for r in range(R):
        lo, hi = D.shard_bounds(n, r, R)
        dev.stein_partial(_lib.FCB_FP64, Xd, lo, hi - lo, scores, hstat, parts[r], None)
    flow, fstat = dev.zeros((n, d)), dev.zeros((8,))
    dev.stein_combine(Xd, R, parts, hstat, flow, fstat, None, 0, None, 0.0)
    ref, _, _ = O.stein_flow(X, q, 0.02, workers=os.cpu_count() or 1)
    assert rel_inf(flow.cpu().numpy(), ref) <= 1e-10
    one = fc.stein_flow(X, fq, fc.SteinConfig(bandwidth=0.02, precision="float64")).a
    assert rel_inf(flow.cpu().numpy(), one) <= 1e-10


@pytest.mark.parametrize("tag,model,method,eta,iters,T", [
    ("ac_sk32", "aircraft_3d", "sinkhorn", 120.0, 15, 800),
    ("ac_st32", "aircraft_3d", "stein", 0.1, 10, 1100),
])
def test_sharded_plan_world1_vs_reference(group1, tag, model, method, eta, iters, T):
    """plan_detailed(group=...) (the multi-GPU code path) on one rank against the
    reference's golden plans, and against the unsharded device planner."""
    g = load_golden("plan_fp32_cases.npz")
    m = fc.get_model(model)
    q = fc.benchmark_mixture(m.workspace_dim)
    tg = fc.SamplePoints(q.sample(2000, [0, STREAM_REFERENCE])) if method == "sinkhorn" else q
    cfg = fc.PlanConfig(method=method, eta=eta, max_iterations=iters, convergence_tol=0.0,
                        metric_interval=0, seed=0)
    disc = fc.Discretization(0.05, T, fc.default_start(m))
    run = fc.plan_detailed(m, tg, disc, cfg, group=group1)
    res = run.result
    assert res.iterations_used == iters
    assert rel_inf(res.trajectory.S, g[f"{tag}_S"]) <= 0.01
    assert rel_inf(res.lqr_costs, g[f"{tag}_lqr_costs"]) <= 0.01
    one = fc.plan_detailed(m, tg, disc, cfg)
    assert rel_inf(res.trajectory.S, one.result.trajectory.S) <= 1e-3
    if method == "sinkhorn":
        # two fp32 kernel paths: a stop test near tol may flip by an iteration
        # late in the plan (up to ~160 inner iterations here)
        assert np.abs(run.flow_log[:, 1:3] - one.flow_log[:, 1:3]).max() <= 3
        assert np.array_equal(run.flow_log[:5, 1:3], one.flow_log[:5, 1:3])


def test_plan_batch_single_rank():
    m = fc.single_integrator_2d()
    q = fc.benchmark_mixture(2)
    probs = [(m, q, fc.Discretization(0.05, 100, np.array([0.1, 0.1])),
              fc.PlanConfig(method="sinkhorn", eta=15.0, max_iterations=3, metric_interval=0,
                            seed=s)) for s in range(3)]
    out = D.plan_batch(probs)
    for s, res in enumerate(out):
        one = fc.plan(*probs[s])
        assert np.array_equal(res.trajectory.S, one.trajectory.S)


@pytest.mark.parametrize("n,d", [(2, 2), (701, 2), (1500, 3)])
def test_sharded_median_tiles_R3_equal_exact_median(n, d):
    """fcb_median_shard_*: three tile ranges histogrammed into one state (what
    the all_reduce sums on a multi-GPU run) select the exact median."""
    import math

    from paper_2511_11514_b200 import _dev

    X = O.benchmark_mixture(d).sample(n, [43, d])
    dev = D.DeviceOps()
    lib = dev.lib
    Xd = dev.tensor(X)
    ws = dev.workspace(lib.fcb_median_workspace_bytes(n), "t_med")
    ntiles = int(lib.fcb_median_tiles(n))
    hstat = dev.zeros((4,))
    s = _dev.stream()
    dev._call("fcb_median_shard_init", n, _dev.ptr(ws), ws.numel(), None, s)
    for p in range(6):
        for r in range(3):
            lo, hi = D.shard_bounds(ntiles, r, 3)
            dev._call("fcb_median_shard_pass", _dev.ptr(Xd), n, d, p, lo, hi, _dev.ptr(ws), None, s)
        dev._call("fcb_median_shard_select", n, p, _dev.ptr(ws), None, s)
    dev._call("fcb_median_shard_finish", n, math.log(n + 1.0), _dev.ptr(hstat), _dev.ptr(ws),
              None, s)
    assert float(hstat[0]) == O.median_bandwidth(X) == fc.median_bandwidth(X)


@pytest.mark.parametrize("method", ["sinkhorn", "stein"])
def test_forced_nccl_collectives_world1_bit_identical(group1, monkeypatch, method):
    """FCB_FORCE_COLLECTIVES=1 issues the NCCL all_gather / all_reduce calls of
    the sharded schedule on the one-rank group (identity operations), so the
    ordering between NCCL's stream and the device steps on the current stream
    is exercised on one GPU: the plan must be bit-identical to the local-copy
    run (a missing wait would read stale gathered buffers)."""
    m = fc.aircraft_3d()
    q = fc.benchmark_mixture(3)
    tg = fc.SamplePoints(q.sample(3000, [0, STREAM_REFERENCE])) if method == "sinkhorn" else q
    cfg = fc.PlanConfig(method=method, eta=120.0 if method == "sinkhorn" else 0.1,
                        max_iterations=4, convergence_tol=0.0, metric_interval=0, seed=0)
    disc = fc.Discretization(0.05, 1500, fc.default_start(m))
    a = fc.plan_detailed(m, tg, disc, cfg, group=group1)
    monkeypatch.setenv("FCB_FORCE_COLLECTIVES", "1")
    b = fc.plan_detailed(m, tg, disc, cfg, group=group1)
    np.testing.assert_array_equal(a.result.trajectory.S, b.result.trajectory.S)
    np.testing.assert_array_equal(a.flow_log, b.flow_log)
