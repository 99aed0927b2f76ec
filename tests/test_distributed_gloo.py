"""Multi-process logic of the M-sharded Sinkhorn flow, world_size 2, gloo, CPU.

The per-shard sweep is injected from the CPU oracle so the collective logic
(all_gather of partial LSEs, fixed-order merge, replicated error and branch,
barycentre combine, global omega) is exercised exactly as on the GPU path.
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


def oracle_sweep(R, S, pot, omega, with_bary):
    Rn, Sn, pn = R.numpy(), S.numpy(), pot.numpy()
    L = O.lse_sweep(Rn, Sn, pn, omega)
    bary = None
    if with_bary:
        w = np.exp((pn[None, :] - O.sqdist(Rn, Sn)) / omega - L[:, None])
        bary = torch.from_numpy(w @ Sn)
    return torch.from_numpy(L), bary


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, X, Y, omega, tol, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_11514_b200 import SinkhornConfig
    from paper_2511_11514_b200.distributed import ShardedSinkhornFlow, shard_rows

    cfg = SinkhornConfig(omega=omega, tol=tol, max_iters=5000)
    flow = ShardedSinkhornFlow(shard_rows(Y, rank, world), cfg, group=dist.group.WORLD,
                               sweep=oracle_sweep, device=torch.device("cpu"))
    a1 = flow(X)
    a2 = flow(X + 1e-3)  # warm-started second call
    np.save(os.path.join(out_dir, f"r{rank}_a1.npy"), a1.a)
    np.save(os.path.join(out_dir, f"r{rank}_a2.npy"), a2.a)
    dist.destroy_process_group()


@pytest.mark.parametrize("omega", ["auto", 0.05])
def test_two_rank_sharded_flow_matches_single_process(tmp_path, omega):
    rng = np.random.default_rng(7)
    X, Y = rng.random((60, 2)), rng.random((97, 2))
    tol = 1e-9
    mp.spawn(_worker, args=(2, _free_port(), X, Y, omega, tol, str(tmp_path)), nprocs=2,
             join=True)
    r0a1, r1a1 = np.load(tmp_path / "r0_a1.npy"), np.load(tmp_path / "r1_a1.npy")
    assert np.array_equal(r0a1, r1a1)  # replicated state: ranks agree bit-for-bit
    warm: dict = {}
    ref1, _, _ = O.sinkhorn_flow(X, Y, omega, 5000, tol, warm)
    ref2, _, _ = O.sinkhorn_flow(X + 1e-3, Y, omega, 5000, tol, warm)
    den = np.abs(ref1).max()
    assert np.abs(r0a1 - ref1).max() / den <= 1e-9
    assert np.abs(np.load(tmp_path / "r0_a2.npy") - ref2).max() / np.abs(ref2).max() <= 1e-9


def test_lse_merge_is_order_fixed_and_exact():
    from paper_2511_11514_b200.distributed import lse_merge

    rng = np.random.default_rng(1)
    full = rng.normal(size=(3, 50)) * 30
    parts = [torch.from_numpy(full[r]) for r in range(3)]
    L, w = lse_merge(parts)
    ref = np.log(np.exp(full - full.max(0)).sum(0)) + full.max(0)
    assert np.allclose(L.numpy(), ref, rtol=1e-14)
    assert np.allclose(sum(x.numpy() for x in w), 1.0)


def test_shard_rows_partitions():
    from paper_2511_11514_b200.distributed import shard_rows

    Y = np.arange(23)[:, None].astype(float)
    parts = [shard_rows(Y, r, 4) for r in range(4)]
    assert np.array_equal(np.concatenate(parts), Y)
    assert max(p.shape[0] for p in parts) - min(p.shape[0] for p in parts) <= 1
