"""Per-rank device time of the M-sharded config-4 flows, measured on ONE GPU.

    python scripts/shard_projection.py [R ...]

Only one GPU is available to this build, so the multi-GPU scaling of the
sharded planner is not measured.  This script measures what one rank of an
R-GPU run executes: the real kernels of distributed.ShardedSinkhorn /
ShardedStein on rank 0's shard (M / R reference samples, T / R self-term rows,
n / R SVGD sources), with a stand-in for the collectives that replicates the
local buffer R times (the merge kernels then process R partials, as on R
ranks).  Inner iteration counts are pinned at 2 (config 4 runs 2 cross and
2-3 self iterations) so every R does the same algorithmic work.  The NCCL transfers are not
included: per inner iteration an all_gather of n (d+1) doubles (3.2 MB at
config 4, ~10 us over NVLink 5).  Rollout and LQR are replicated on every rank
and timed separately.  The output is a PROJECTION, labelled as such.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_11514_b200 as fc  # noqa: E402
from paper_2511_11514_b200 import distributed as D  # noqa: E402


class ReplicatedCollectives:
    """rank 0 of `world`, every other rank assumed to hold the same data."""

    def __init__(self, world):
        self.rank, self.world, self.group = 0, world, None

    def all_gather(self, out, inp):
        flat = inp.reshape(-1)
        out.view(self.world, -1).copy_(flat.unsqueeze(0).expand(self.world, -1))

    def all_reduce_sum(self, t):
        t.mul_(self.world)
        return t


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    Rs = [int(v) for v in sys.argv[1:]] or [1, 2, 4, 8]
    T, M, d = 100_000, 1_000_000, 3
    m = fc.aircraft_3d()
    cfg = fc.PlanConfig(method="sinkhorn", seed=0)
    S = fc.rollout(m, fc.default_start(m), fc.initial_controls(cfg, m, T), 0.05)
    X = torch.from_numpy(np.ascontiguousarray(m.project_states(S[1:]))).cuda()
    Y = fc.benchmark_mixture(3).sample(M, [0, 2])
    q3 = fc.benchmark_mixture(3)
    rows = []
    for R in Rs:
        coll = ReplicatedCollectives(R)
        sk_cfg = fc.SinkhornConfig(max_iters=2, tol=1e-30, precision="float32")
        sk = D.ShardedSinkhorn(D.shard_rows(Y, 0, R), T, sk_cfg)
        sk.coll = coll
        # re-derive the quantities the constructor took from the real collectives
        sk.ysum.mul_(R)
        sk.m_global = sk.Y.shape[0] * R
        sk.logb = -np.log(sk.m_global)
        sk.log_frac = np.log(1.0 / R)
        sk.rows = D.shard_bounds(T, 0, R)
        sk.nown = sk.rows[1] - sk.rows[0]
        sk.chunk = (T + R - 1) // R
        z = lambda *s: torch.zeros(s, dtype=torch.float64, device="cuda")  # noqa: E731
        sk.gath_x, sk.gath_s = z(R, T, d + 1), z(R, sk.chunk, d + 4)
        sk.Lb, sk.send_s = z(sk.nown, d + 1), z(sk.chunk, d + 4)
        wf, wp, wv = z(T), z(T), torch.zeros(2, dtype=torch.int32, device="cuda")
        flow, fstat = z(T, d), z(8)

        def sinkhorn_flow():
            sk.flow_into(X, wf, wp, wv, flow, fstat)

        t_sk = timed(sinkhorn_flow)
        it = (int(fstat[5]), int(fstat[6]))
        sv = D.ShardedStein(T, d, q3, 0.01)
        sv.coll = coll
        sv.cols = D.shard_bounds(T, 0, R)
        sv.parts = z(R, T, d + 1)
        t_sv = timed(lambda: sv.flow_into(X, flow, fstat))
        rows.append({"R": R, "sinkhorn_flow_ms": t_sk, "inner_iterations": it,
                     "svgd_flow_ms": t_sv})
        print(json.dumps(rows[-1]), flush=True)
    base = rows[0]
    out = {"what": "per-rank device time of the sharded config-4 flows (rank 0's shard, one GPU, "
                   "collectives replaced by replication; NCCL transfers excluded) -- a projection",
           "rows": rows,
           "flow_speedup_vs_R1": {r["R"]: (base["sinkhorn_flow_ms"] + base["svgd_flow_ms"])
                                  / (r["sinkhorn_flow_ms"] + r["svgd_flow_ms"]) for r in rows}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
