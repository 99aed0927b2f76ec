"""Sharded Sinkhorn flow and batched planning with the CUDA sweep (one GPU).

The multi-rank collective logic is covered on CPU by test_distributed_gloo;
here the device sweep (FCB_OT_SWEEP with barycentres) drives the same host
algorithm, shards emulated in one process by merging per-shard sweeps.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2511_11514_b200 as fc
from fcb_testutil import rel_inf
from oracle import flowcover_oracle as O
from paper_2511_11514_b200 import distributed as D

pytestmark = pytest.mark.gpu


def test_sharded_flow_single_rank_matches_unsharded():
    rng = np.random.default_rng(3)
    X, Y = rng.random((1500, 2)), rng.random((6000, 2))
    cfg = fc.SinkhornConfig()
    flow = D.ShardedSinkhornFlow(Y, cfg)
    a = flow(X).a
    ref = fc.sinkhorn_flow(X, fc.SamplePoints(Y), cfg).a
    assert rel_inf(a, ref) <= 1e-4


@pytest.mark.parametrize("precision", ["float32", "float64"])
def test_device_sweep_shards_merge_to_the_full_sweep(precision):
    """Emulate 4 shards: per-shard device sweeps merged by lse_merge."""
    rng = np.random.default_rng(5)
    X = torch.from_numpy(rng.random((700, 3))).cuda()
    Y = rng.random((4000, 3))
    pot = torch.from_numpy(rng.normal(scale=0.01, size=4000)).cuda()
    sweep = D.cuda_sweep(precision)
    Ls, bs = [], []
    for r in range(4):
        lo, hi = 1000 * r, 1000 * (r + 1)
        L, b = sweep(X, torch.from_numpy(Y[lo:hi]).cuda(), pot[lo:hi].contiguous(), 0.03, True)
        Ls.append(L)
        bs.append(b)
    L, w = D.lse_merge(Ls)
    ybar = sum(wi[:, None] * bi for wi, bi in zip(w, bs))
    Lref = O.lse_sweep(X.cpu().numpy(), Y, pot.cpu().numpy(), 0.03)
    wref = np.exp((pot.cpu().numpy()[None, :] - O.sqdist(X.cpu().numpy(), Y)) / 0.03 - Lref[:, None])
    tol = 1e-5 if precision == "float32" else 1e-12
    assert rel_inf(L.cpu().numpy(), Lref) <= tol
    assert rel_inf(ybar.cpu().numpy(), wref @ Y) <= tol


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
