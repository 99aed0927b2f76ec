"""The sharded flows' collective schedule at world sizes 2 and 4 (gloo, CPU).

distributed.ShardedSinkhorn / ShardedStein run with the CPU stand-in of the
device steps (tests/shard_cpu_ops.py) and torch.distributed gloo collectives:
reference samples (Sinkhorn) or SVGD sources sharded over the ranks, partial
LSEs / kernel sums all-gathered and merged in rank order, loop control on
replicated words.  Checked against the single-process oracle (the reference's
algorithm): flows, warm potentials, inner iteration counts, and whole planner
runs; every rank must hold bit-identical results.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from fcb_testutil import ROOT  # noqa: F401  (puts the repo on sys.path)
from oracle import flowcover_oracle as O


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _sinkhorn_worker(rank, world, port, X, Y, omega, tol, out_dir):
    _init(rank, world, port)
    from shard_cpu_ops import CpuOps

    from paper_2511_11514_b200 import SinkhornConfig
    from paper_2511_11514_b200.distributed import ShardedSinkhornFlow, shard_rows

    cfg = SinkhornConfig(omega=omega, tol=tol, max_iters=5000)
    flow = ShardedSinkhornFlow(shard_rows(Y, rank, world), cfg, group=dist.group.WORLD,
                               ops=CpuOps())
    st1, st2 = {}, {}
    a1 = flow(X, stats=st1)
    a2 = flow(X + 1e-3, stats=st2)  # warm-started second call
    wf, wp, _ = flow.warm
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), a1=a1.a, a2=a2.a, f=wf.numpy(), p=wp.numpy(),
             inner=np.array([st1["iters_cross"], st1["iters_self"], st2["iters_cross"],
                             st2["iters_self"]]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("omega", ["auto", 0.05])
def test_sharded_sinkhorn_flow_matches_single_process(tmp_path, world, omega):
    rng = np.random.default_rng(7)
    X, Y = rng.random((60, 2)), rng.random((97, 2))
    tol = 1e-9
    mp.spawn(_sinkhorn_worker, args=(world, _free_port(), X, Y, omega, tol, str(tmp_path)),
             nprocs=world, join=True)
    res = [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]
    for r in range(1, world):  # replicated state: ranks agree bit for bit
        for k in ("a1", "a2", "f", "p", "inner"):
            assert np.array_equal(res[0][k], res[r][k]), (r, k)
    warm: dict = {}
    s1, s2 = {}, {}
    ref1, _, _ = O.sinkhorn_flow(X, Y, omega, 5000, tol, warm, stats=s1)
    ref2, _, _ = O.sinkhorn_flow(X + 1e-3, Y, omega, 5000, tol, warm, stats=s2)
    assert list(res[0]["inner"]) == [s1["iters_cross"], s1["iters_self"], s2["iters_cross"],
                                     s2["iters_self"]]
    assert np.abs(res[0]["a1"] - ref1).max() / np.abs(ref1).max() <= 1e-9
    assert np.abs(res[0]["a2"] - ref2).max() / np.abs(ref2).max() <= 1e-9
    assert np.abs(res[0]["f"] - warm["f"]).max() / np.abs(warm["f"]).max() <= 1e-9
    assert np.abs(res[0]["p"] - warm["p"]).max() / np.abs(warm["p"]).max() <= 1e-9


def _stein_worker(rank, world, port, X, bandwidth, out_dir):
    _init(rank, world, port)
    from shard_cpu_ops import CpuOps

    from paper_2511_11514_b200.distributed import ShardedStein

    n, d = X.shape
    ops = CpuOps()
    sv = ShardedStein(n, d, O.benchmark_mixture(d), bandwidth, group=dist.group.WORLD, ops=ops)
    flow, fstat = torch.zeros((n, d), dtype=torch.float64), torch.zeros(8, dtype=torch.float64)
    sv.flow_into(torch.from_numpy(X), flow, fstat)
    np.savez(os.path.join(out_dir, f"s{rank}.npz"), a=flow.numpy(), fstat=fstat.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("bandwidth", ["median", 0.02])
def test_sharded_stein_matches_single_process(tmp_path, world, bandwidth):
    rng = np.random.default_rng(9)
    X = rng.normal(0.5, 0.2, size=(83, 3))
    mp.spawn(_stein_worker, args=(world, _free_port(), X, bandwidth, str(tmp_path)), nprocs=world,
             join=True)
    res = [dict(np.load(tmp_path / f"s{r}.npz")) for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(res[0]["a"], res[r]["a"])
    ref, h, _ = O.stein_flow(X, O.benchmark_mixture(3), bandwidth)
    assert res[0]["fstat"][4] == pytest.approx(h, rel=1e-14)
    assert np.abs(res[0]["a"] - ref).max() / np.abs(ref).max() <= 1e-12


# ---- whole planner runs with the sharded flows ----------------------------------
def sharded_oracle_plan(model, s0, dt, T, method, eta, iterations, group, ops, targets=None,
                        q=None, bandwidth="median"):
    """O.plan (optimizer.py:221-269) with the flow evaluated by the sharded
    schedule: the loop plan_detailed(group=...) runs on the GPU, here with the
    oracle's rollout / LQR and the CPU stand-in of the device steps."""
    from paper_2511_11514_b200 import SinkhornConfig
    from paper_2511_11514_b200.distributed import ShardedSinkhorn, ShardedStein, shard_rows

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    f, ja, jb, P = O.model_fns(model)
    m = 3 if model == "aircraft_3d" else 2
    rng = np.random.default_rng(np.random.SeedSequence([0, 1]))
    U = 1e-2 * rng.standard_normal((T, m))
    d = P.shape[0]
    Qw, Rw = P.T @ P, 0.1 * np.eye(m)
    if method == "sinkhorn":
        fl = ShardedSinkhorn(shard_rows(targets, rank, world), T, SinkhornConfig(), group, ops)
    else:
        fl = ShardedStein(T, d, q, bandwidth, group, ops)
    z = lambda *s: torch.zeros(s, dtype=torch.float64)  # noqa: E731
    wf, wp, wv = z(T), z(T), torch.zeros(2, dtype=torch.int32)
    state = torch.zeros(8, dtype=torch.int32)
    log = z(iterations, 4)
    norms = []
    for it in range(iterations):
        S, fail = O.rollout(f, s0, U, dt)
        assert fail < 0
        X = torch.from_numpy(np.ascontiguousarray(S[1:] @ P.T))
        flow, fstat = z(T, d), z(8)
        if method == "sinkhorn":
            fl.flow_into(X, wf, wp, wv, flow, fstat, state, it, log, 0.0)
        else:
            fl.flow_into(X, flow, fstat, state, it, log, 0.0)
        a = flow.numpy()
        norms.append(float(log[it, 0]))
        A, B = O.linearize(ja, jb, S, U)
        sol = O.solve_flow_lqr(A, B, dt, a @ P, Qw, Rw)
        U = U + eta * sol["v"]
    S, _ = O.rollout(f, s0, U, dt)
    return S, np.array(norms), log.numpy()


def _plan_worker(rank, world, port, case, out_dir):
    _init(rank, world, port)
    from shard_cpu_ops import CpuOps

    ops = CpuOps()
    model, s0, T, method, eta, iters = case
    d = 3 if model == "aircraft_3d" else 2
    q = O.benchmark_mixture(d)
    targets = q.sample(150, [0, 2]) if method == "sinkhorn" else None
    S, norms, log = sharded_oracle_plan(model, np.array(s0), 0.05, T, method, eta, iters,
                                        dist.group.WORLD, ops, targets=targets, q=q)
    np.savez(os.path.join(out_dir, f"p{rank}.npz"), S=S, norms=norms, log=log)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", [
    ("single_integrator_2d", [0.1, 0.1], 40, "sinkhorn", 6.0, 4),
    ("double_integrator_2d", [0.1, 0.1, 0.0, 0.0], 40, "stein", 0.1, 4),
])
def test_sharded_plan_matches_single_process_oracle(tmp_path, world, case):
    mp.spawn(_plan_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world,
             join=True)
    res = [dict(np.load(tmp_path / f"p{r}.npz")) for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(res[0]["S"], res[r]["S"])
    model, s0, T, method, eta, iters = case
    d = 2
    q = O.benchmark_mixture(d)
    kw = dict(targets=q.sample(150, [0, 2])) if method == "sinkhorn" else dict(q=q)
    ref = O.plan(model, np.array(s0), 0.05, T, method, eta, iters, **kw)
    assert np.abs(res[0]["S"] - ref["S"]).max() / np.abs(ref["S"]).max() <= 1e-9
    # SVGD sums centred on X[0] and merged across shards: ~1e-8 relative rounding
    # (the (2/h) x terms cancel), far inside the north_star's 1e-4
    np.testing.assert_allclose(res[0]["norms"], ref["flow_norms"],
                               rtol=1e-9 if method == "sinkhorn" else 1e-6)
    if method == "sinkhorn":
        assert [tuple(int(v) for v in row[1:3]) for row in res[0]["log"]] == \
            [tuple(x) for x in ref["inner"]]


def test_shard_bounds_partition():
    from paper_2511_11514_b200.distributed import shard_bounds, shard_rows

    Y = np.arange(23)[:, None].astype(float)
    parts = [shard_rows(Y, r, 4) for r in range(4)]
    assert np.array_equal(np.concatenate(parts), Y)
    assert max(p.shape[0] for p in parts) - min(p.shape[0] for p in parts) <= 1
    assert [shard_bounds(23, r, 4) for r in range(4)] == [(0, 5), (5, 11), (11, 17), (17, 23)]


def _uneven_worker(rank, world, port, X, Y, out_dir):
    _init(rank, world, port)
    from shard_cpu_ops import CpuOps

    from paper_2511_11514_b200 import FlowError, SinkhornConfig
    from paper_2511_11514_b200.distributed import ShardedSinkhornFlow, shard_rows

    flow = ShardedSinkhornFlow(shard_rows(Y, rank, world),
                               SinkhornConfig(omega=0.03, tol=1e-10, max_iters=5000),
                               group=dist.group.WORLD, ops=CpuOps())
    st: dict = {}
    a = flow(X, stats=st)
    # an iteration budget too small for the tolerance: every rank raises FlowError
    tight = ShardedSinkhornFlow(shard_rows(Y, rank, world),
                                SinkhornConfig(omega=0.03, tol=1e-12, max_iters=2),
                                group=dist.group.WORLD, ops=CpuOps())
    raised = False
    try:
        tight(X)
    except FlowError:
        raised = True
    np.savez(os.path.join(out_dir, f"u{rank}.npz"), a=a.a, raised=np.array(raised),
             inner=np.array([st["iters_cross"], st["iters_self"]]))
    dist.destroy_process_group()


def test_three_ranks_uneven_shards_and_flow_error(tmp_path):
    """world 3: neither n = 50 nor m = 101 divides evenly (shards of 16/17 self
    rows and 33/34 samples); the budget-starved solve raises FlowError on every
    rank, as sinkhorn.py:370-373 does."""
    rng = np.random.default_rng(11)
    X, Y = rng.random((50, 2)), rng.random((101, 2))
    mp.spawn(_uneven_worker, args=(3, _free_port(), X, Y, str(tmp_path)), nprocs=3, join=True)
    res = [dict(np.load(tmp_path / f"u{r}.npz")) for r in range(3)]
    for r in range(1, 3):
        assert np.array_equal(res[0]["a"], res[r]["a"])
    assert all(bool(r["raised"]) for r in res)
    st: dict = {}
    ref, _, _ = O.sinkhorn_flow(X, Y, 0.03, 5000, 1e-10, stats=st)
    assert list(res[0]["inner"]) == [st["iters_cross"], st["iters_self"]]
    assert np.abs(res[0]["a"] - ref).max() / np.abs(ref).max() <= 1e-9
