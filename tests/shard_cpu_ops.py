"""CPU stand-in for the device steps of the sharded flows -- TEST INFRASTRUCTURE.

Implements the methods of paper_2511_11514_b200.distributed.DeviceOps with
torch CPU tensors and the oracle's sweeps, following the kernels of
csrc/shard.cu step for step (gating on the loop-control words, fixed-order
merges, last-iteration outputs).  With it the collective schedule of
ShardedSinkhorn / ShardedStein runs under the gloo backend on CPU, at world
sizes > 1, against the single-process oracle.  The CUDA kernels themselves
are checked against the oracle by the -m gpu tests.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from oracle import flowcover_oracle as O

EXP_CLIP = 500.0


class _Done:
    def synchronize(self):
        return None


class CpuOps:
    def zeros(self, shape, dtype=torch.float64):
        return torch.zeros(shape, dtype=dtype)

    def tensor(self, a):
        return torch.from_numpy(np.array(a, dtype=np.float64, copy=True, order="C"))

    def snapshot(self, src, dst):
        dst.copy_(src)
        return _Done()

    def pinned_int(self):
        return torch.zeros(1, dtype=torch.int32)

    # ---- Sinkhorn ----------------------------------------------------------
    def point_sums(self, P, out):
        d = P.shape[1]
        out[:d] = P.sum(dim=0)
        out[d] = (P * P).sum()
        out[d + 1] = float(P.shape[0])

    def lse_sweep(self, prec, R, S, scal, pot, scale, shift, out, bary, gate, tag, est=None,
                  est_logw=0.0):
        if gate is not None and int(gate[0]) != 0:
            return
        w = float(scal[0])
        Rn, Sn, pn = R.numpy(), S.numpy(), pot.numpy()
        L = O.lse_sweep(Rn, Sn, pn, w)
        if out is not None:
            out.copy_(torch.from_numpy(scale * w * (shift - L) if scale != 0.0 else L))
        if bary is not None:
            wts = np.exp((pn[None, :] - O.sqdist(Rn, Sn)) / w - L[:, None])
            bary[:, 0] = torch.from_numpy(L)
            bary[:, 1:] = torch.from_numpy(wts @ Sn)

    def shard_init(self, prec, X, ysum, omega_fixed, warm_f, warm_p, warm_valid, scal_x, scal_s,
                   f, p, ctl, eslot, plan_state):
        n, d = X.shape
        skip = plan_state is not None and int(plan_state[0]) != 0
        mx = X.mean(dim=0)
        m = float(ysum[d + 1])
        my = ysum[:d] / m
        if omega_fixed > 0:
            w = omega_fixed
        else:
            msq = float((X * X).sum(dim=1).mean() + ysum[d] / m - 2.0 * (mx @ my))
            w = max(0.05 * msq, 1e-12)
        scal_x.zero_()
        scal_s.zero_()
        scal_x[0] = scal_s[0] = w
        ctl.zero_()
        ctl[0] = ctl[1] = ctl[7] = int(skip)
        eslot.zero_()
        vf = warm_valid is not None and int(warm_valid[0]) != 0
        vp = warm_valid is not None and int(warm_valid[1]) != 0
        f.copy_(warm_f if vf else torch.zeros(n, dtype=torch.float64))
        p.copy_(warm_p if vp else torch.zeros(n, dtype=torch.float64))

    def cross_merge(self, n, d, R, gath, scal, tol, max_iters, f, fnext, rs, mass, ybar, ctl,
                    eslot, stat):
        if int(ctl[0]) != 0:
            return
        w = float(scal[0])
        loga = -math.log(n)
        Ls = gath[:, :, 0]  # (R, n)
        M = Ls.max(dim=0).values
        M = torch.where(torch.isfinite(M), M, torch.zeros_like(M))
        e = torch.exp(Ls - M)
        S = e.sum(dim=0)
        L = M + torch.log(S)
        A = (e[:, :, None] * gath[:, :, 1:]).sum(dim=0)
        upd = w * (loga - L)
        delta = torch.clamp((f - upd) / w, max=EXP_CLIP)
        err = float(torch.abs(torch.expm1(delta)).max()) / n
        rs.copy_(torch.exp(delta + loga))
        mass.copy_(torch.exp(f / w + L))
        ybar.copy_(A / S[:, None])
        fnext.copy_(upd)
        it = int(ctl[2]) + 1
        ctl[2] = it
        conv = err <= tol
        if conv or it >= max_iters:
            stat.copy_(torch.tensor([err, float(it), float(conv), 0.0], dtype=torch.float64))
            ctl[0] = 1
        else:
            f.copy_(fnext)

    def self_rows(self, n, d, row0, nown, Lb, scal, p, send, ctl):
        if int(ctl[1]) != 0:
            return
        w = float(scal[0])
        loga = -math.log(n)
        L = Lb[:nown, 0]
        pi = p[row0:row0 + nown]
        target = w * (loga - L)
        delta = torch.clamp((pi - target) / w, max=EXP_CLIP)
        send[:nown, 0] = 0.5 * (pi + target)
        send[:nown, 1] = torch.exp(delta + loga)
        send[:nown, 2] = torch.exp(pi / w + L)
        send[:nown, 3] = torch.abs(torch.expm1(delta))
        send[:nown, 4:] = Lb[:nown, 1:]

    def self_commit(self, n, d, R, chunk, gath, tol, max_iters, p, pnext, rho, massp, xbar, ctl,
                    eslot, stat):
        if int(ctl[1]) != 0:
            return
        rows = []
        for r in range(R):
            lo, hi = (n * r) // R, (n * (r + 1)) // R
            rows.append(gath[r, : hi - lo])
        allr = torch.cat(rows)
        pnext.copy_(allr[:, 0])
        rho.copy_(allr[:, 1])
        massp.copy_(allr[:, 2])
        xbar.copy_(allr[:, 4:])
        err = float(allr[:, 3].max()) / n
        it = int(ctl[3]) + 1
        ctl[3] = it
        conv = err <= tol
        if conv or it >= max_iters:
            stat.copy_(torch.tensor([err, float(it), float(conv), 0.0], dtype=torch.float64))
            ctl[1] = 1
        else:
            p.copy_(pnext)

    def flow_finish(self, X, rs, mass, ybar, rho, massp, xbar, stat_x, stat_p, tol, f, p, warm_f,
                    warm_p, warm_valid, flow, fstat, scal, plan_state, iteration, flow_log,
                    conv_tol, ctl):
        if int(ctl[7]) != 0:
            return
        worst = max(float(stat_x[0]), float(stat_p[0]))
        flow_error = worst > 100.0 * tol
        mean_mag = float("nan")
        if not flow_error:
            grad = (2.0 * (rs[:, None] * X - mass[:, None] * ybar)
                    - 2.0 * (rho[:, None] * X - massp[:, None] * xbar))
            flow.copy_(-grad)
            mean_mag = float(torch.sqrt((grad * grad).sum(dim=1)).sum()) / X.shape[0]
            if warm_f is not None:
                warm_f.copy_(f)
                warm_p.copy_(p)
                warm_valid[0] = warm_valid[1] = 1
        fstat.copy_(torch.tensor([worst, float(stat_x[2] != 0 and stat_p[2] != 0),
                                  float(flow_error), mean_mag, float(scal[0]), float(stat_x[1]),
                                  float(stat_p[1]), 0.0], dtype=torch.float64))
        if plan_state is not None:
            if flow_error:
                plan_state[0], plan_state[1], plan_state[2], plan_state[3] = 2, 2, iteration, -1
            else:
                flow_log[iteration] = torch.tensor([mean_mag, fstat[5], fstat[6], worst])
                plan_state[4] = iteration + 1
                if mean_mag < conv_tol:
                    plan_state[0] = 1

    # ---- SVGD ---------------------------------------------------------------
    def mixture_params(self, q):
        self.mixture = q  # an oracle Mixture: .score on host arrays
        return q.mu.shape[0], None

    def median_bandwidth(self, X, hstat, gate):
        if gate is not None and int(gate[0]) != 0:
            return
        Xn = X.numpy()
        h = O.median_bandwidth(Xn)
        med = math.sqrt(h * math.log(Xn.shape[0] + 1.0))
        clamped = h <= 1e-12
        hstat.copy_(torch.tensor([max(h, 1e-12), med, float(clamped), 0.0], dtype=torch.float64))

    def median_sharded(self, X, hstat, gate, coll):
        """The radix selection of csrc/stein.cu over this rank's 64 x 64 pair tiles
        (upper triangle, i < j, each pair counted twice, the n diagonal zeros
        added in the first bucket), histograms all-reduced per pass."""
        if gate is not None and int(gate[0]) != 0:
            return
        Xn = X.numpy()
        n = Xn.shape[0]
        nb = (n + 63) // 64
        tiles = [(bi, bj) for bi in range(nb) for bj in range(bi, nb)]
        lo, hi = (len(tiles) * coll.rank) // coll.world, (len(tiles) * (coll.rank + 1)) // coll.world
        keys = []
        for bi, bj in tiles[lo:hi]:
            I = np.arange(bi * 64, min(n, bi * 64 + 64))
            J = np.arange(bj * 64, min(n, bj * 64 + 64))
            d2 = O.sqdist(Xn[I], Xn[J])
            keep = J[None, :] > I[:, None]
            keys.append(d2[keep])
        keys = np.concatenate(keys).view(np.uint64) if keys else np.zeros(0, np.uint64)
        N = n * n
        prefix, rank = [0, 0], [(N - 1) // 2, N // 2]
        for shift, bits in zip((52, 41, 30, 19, 8, 0), (11, 11, 11, 11, 11, 8)):
            hshift = shift + bits
            same = prefix[0] == prefix[1]
            hist = np.zeros((2, 2048), dtype=np.int64)
            hi_bits = keys >> np.uint64(hshift) if hshift < 64 else np.zeros_like(keys)
            dig = ((keys >> np.uint64(shift)) & np.uint64((1 << bits) - 1)).astype(np.int64)
            for t in (0,) if same else (0, 1):
                sel = hi_bits == np.uint64(prefix[t])
                hist[t] += 2 * np.bincount(dig[sel], minlength=2048)
            h = torch.from_numpy(hist)
            coll.all_reduce_sum(h)
            hist = h.numpy()
            for t in (0, 1):
                hh = hist[0 if same else t].copy()
                if prefix[t] == 0:
                    hh[0] += n
                csum = np.cumsum(hh)
                b = int(np.searchsorted(csum, rank[t], side="right"))
                rank[t] -= int(csum[b - 1]) if b > 0 else 0
                prefix[t] = (prefix[t] << bits) | b
        vlo = np.array([prefix[0]], dtype=np.uint64).view(np.float64)[0]
        vhi = np.array([prefix[1]], dtype=np.uint64).view(np.float64)[0]
        med = math.sqrt(vlo) if N % 2 else (math.sqrt(vlo) + math.sqrt(vhi)) / 2.0
        h = med * med / math.log(n + 1.0)
        clamped = h <= 1e-12
        hstat.copy_(torch.tensor([1e-12 if clamped else h, med, float(clamped), 0.0],
                                 dtype=torch.float64))

    def gmm_score(self, X, k, params, out, gate):
        if gate is not None and int(gate[0]) != 0:
            return
        out.copy_(torch.from_numpy(self.mixture.score(X.numpy())))

    def stein_partial(self, prec, X, col0, ncols, scores, hstat, part, gate):
        if gate is not None and int(gate[0]) != 0:
            return
        h = float(hstat[0])
        Xn = X.numpy()
        c = Xn[0]
        cols = slice(col0, col0 + ncols)
        K = np.exp(-O.sqdist(Xn, Xn[cols]) / h)
        wj = scores.numpy()[cols] - (2.0 / h) * (Xn[cols] - c)
        part[:, 0] = torch.from_numpy(K.sum(axis=1))
        part[:, 1:] = torch.from_numpy(K @ wj)

    def stein_combine(self, X, R, parts, hstat, flow, fstat, plan_state, iteration, flow_log,
                      conv_tol):
        if plan_state is not None and int(plan_state[0]) != 0:
            return
        n = X.shape[0]
        h = float(hstat[0])
        tot = parts.sum(dim=0)
        xc = X - X[0]
        out = (tot[:, 1:] + (2.0 / h) * xc * tot[:, :1]) / n
        flow.copy_(out)
        mean_mag = float(torch.sqrt((out * out).sum(dim=1)).sum()) / n
        if fstat is not None:
            fstat.copy_(torch.tensor([0.0, 1.0, 0.0, mean_mag, h, float(hstat[2]),
                                      float(hstat[1]), 0.0], dtype=torch.float64))
        if plan_state is not None:
            flow_log[iteration] = torch.tensor([mean_mag, h, float(hstat[2]), float(hstat[1])])
            plan_state[4] = iteration + 1
            if mean_mag < conv_tol:
                plan_state[0] = 1
