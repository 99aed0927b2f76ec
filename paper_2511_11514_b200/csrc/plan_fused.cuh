// plan_fused.cuh -- the coverage loop of a linear model in ONE persistent
// launch (optimizer.py:221-269 for iterations it0..maxit-1): per iteration
//
//   rollout    s_{k+1} = Phi s_k + Gam u_k           (affine scan, X = P S)
//   flow       the resident Sinkhorn flow (flow_resident.cuh)
//   LQR        eta backward scan (emits d), z forward scan (v*, cost,
//              U <- clamp(U + eta v*)) on the stored Riccati phase
//
// with grid barriers (grid groups: one problem over every SM) or
// __syncthreads (CTA groups: one problem per CTA, batched) between the
// phases, device-side stop tests and no host round trip.  Included at the end
// of dynamics.cu (needs Model<>, LiftedFlow, phigam_compute).
//
// Affine scans: CTA r of a grid group owns steps [T r/G, T (r+1)/G) -- the
// same rows as its flow slice, so the flow -> LQR -> rollout hand-offs are
// CTA-local; only the scan carries cross CTAs (one barrier per scan).  In a
// CTA, up to 128 threads each compose a run of L consecutive steps, a
// Hillis-Steele scan over the runs in shared memory gives every run its
// prefix, and the grid carry is the same scan over the CTAs' aggregates.
#pragma once

#include "affscan.cuh"
#include "flow_resident.cuh"
#include "plan_scan.cuh"

namespace fcb {

constexpr int PF_RUNS = 128;    // composing threads per CTA scan
constexpr int PF_CARRY = 256;   // max CTAs of a grid group

template <int N>
struct PfSmem {
    AMap<N> run[2][PF_RUNS];    // per-run maps (ping-pong)
    AMap<N> car[2][PF_CARRY];   // CTA aggregates (grid carry)
    double xs[N];               // state at the chunk start
    double red[RS_WARPS];
    int ired[RS_WARPS];
};

template <int N>
constexpr size_t pf_smem_bytes() {
    return sizeof(PfSmem<N>);
}

// in-place inclusive scan over n maps in buf[0] (position order); returns the
// buffer holding the result; every thread of the CTA calls it
template <int N>
__device__ AMap<N>* pf_scan(AMap<N>* a, AMap<N>* b, int n) {
    for (int o = 1; o < n; o <<= 1) {
        for (int i = threadIdx.x; i < n; i += RS_BLOCK) {
            // operands in registers: composing straight out of shared memory
            // re-loads every operand (the compiler cannot rule out aliasing)
            const AMap<N> later = a[i];
            if (i >= o) {
                const AMap<N> earlier = a[i - o];
                AMap<N> r;
                amap_compose(later, earlier, r);
                b[i] = r;
            } else {
                b[i] = later;
            }
        }
        __syncthreads();
        AMap<N>* t = a;
        a = b;
        b = t;
    }
    return a;
}

struct PfChunk {
    int k0, k1;    // steps owned by this CTA
    int p0, cnt;   // positions of the chunk (scan order)
    int c;         // chunk index in scan order
    int L, nact;   // steps per run, runs
};

template <bool FWD, bool GRID>
__device__ __forceinline__ PfChunk pf_chunk(int T, const RsGroup<GRID>& grp) {
    PfChunk ch;
    ch.k0 = (int)((long long)T * grp.rank / grp.size);
    ch.k1 = (int)((long long)T * (grp.rank + 1) / grp.size);
    ch.cnt = ch.k1 - ch.k0;
    ch.p0 = FWD ? ch.k0 : T - ch.k1;
    ch.c = FWD ? grp.rank : grp.size - 1 - grp.rank;
    ch.L = ch.cnt > 0 ? (ch.cnt + PF_RUNS - 1) / PF_RUNS : 1;
    ch.nact = (ch.cnt + ch.L - 1) / ch.L;
    return ch;
}

// Phase 1: the runs' maps, their inclusive scan (kept in shared memory) and
// (grid groups) the chunk aggregate published for the carry.
template <int N, bool FWD, class MapFn>
__device__ AMap<N>* pf_phase1(int T, const PfChunk& ch, const MapFn& mapf, PfSmem<N>& sm,
                              double* agg_pub) {
    const int t = threadIdx.x;
    if (ch.nact <= 32) {
        // one warp: runs in lanes, inclusive scan by shuffles (no block syncs)
        if (t < 32) {
            AMap<N> acc;
            amap_identity(acc);
            if (t < ch.nact) {
                AMap<N> m, tmp;
                const int pa = ch.p0 + t * ch.L, pb = min(pa + ch.L, ch.p0 + ch.cnt);
                for (int p = pa; p < pb; ++p) {
                    mapf(FWD ? p : T - 1 - p, m);
                    amap_compose(m, acc, tmp);
                    acc = tmp;
                }
            }
#pragma unroll 1
            for (int o = 1; o < 32; o <<= 1) {
                AMap<N> prev, tmp;
                amap_shfl(prev, acc, o, true);
                if (t >= o) {
                    amap_compose(acc, prev, tmp);
                    acc = tmp;
                }
            }
            if (t < ch.nact) sm.run[0][t] = acc;
            if (agg_pub && t == max(ch.nact - 1, 0)) {
                if (ch.nact == 0) amap_identity(acc);
                amap_copy_to(agg_pub + (size_t)ch.c * (N * N + N), acc);
            }
        }
        __syncthreads();
        return sm.run[0];
    }
    if (t < ch.nact) {
        AMap<N> acc, m, tmp;
        amap_identity(acc);
        const int pa = ch.p0 + t * ch.L, pb = min(pa + ch.L, ch.p0 + ch.cnt);
        for (int p = pa; p < pb; ++p) {
            mapf(FWD ? p : T - 1 - p, m);
            amap_compose(m, acc, tmp);
            acc = tmp;
        }
        sm.run[0][t] = acc;
    }
    __syncthreads();
    AMap<N>* inc = pf_scan<N>(sm.run[0], sm.run[1], ch.nact);
    if (agg_pub && t == 0) {
        AMap<N> tot;
        if (ch.nact > 0) tot = inc[ch.nact - 1];
        else amap_identity(tot);
        double* dst = agg_pub + (size_t)ch.c * (N * N + N);
        amap_copy_to(dst, tot);
    }
    return inc;
}

// Composition A_{c-1} o ... o A_0 of the first c published chunk aggregates:
// warps load 32 maps each, an ordered shuffle tree (lane i absorbs lane i+o,
// the later map) reduces each warp, thread 0 chains the warp results.
template <int N>
__device__ void pf_carry(const double* agg_pub, int c, PfSmem<N>& sm, AMap<N>& out) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int nw = (c + 31) >> 5;
    if (w < nw) {
        AMap<N> mine;
        const int i = w * 32 + lane;
        if (i < c) amap_copy_from(agg_pub + (size_t)i * (N * N + N), mine);
        else amap_identity(mine);
#pragma unroll 1
        for (int o = 1; o < 32; o <<= 1) {
            AMap<N> later, tmp;
            amap_shfl(later, mine, o, false);
            if ((lane & (2 * o - 1)) == 0) {
                amap_compose(later, mine, tmp);
                mine = tmp;
            }
        }
        if (lane == 0) sm.car[0][w] = mine;
    }
    __syncthreads();
    if (t == 0) {
        AMap<N> acc = sm.car[0][0];
        for (int k = 1; k < nw; ++k) {
            const AMap<N> nxt = sm.car[0][k];
            AMap<N> tmp;
            amap_compose(nxt, acc, tmp);
            acc = tmp;
        }
        out = acc;
    }
}

// Phase 2: the chunk's start state (init carried over the earlier chunks'
// aggregates), then every run steps through its positions calling
// out(k, x_k, x_k+1) (states in scan order).  Returns the thread's sum of out.
template <int N, bool FWD, bool GRID, class MapFn, class OutFn>
__device__ double pf_phase2(int T, const PfChunk& ch, const MapFn& mapf, const OutFn& out,
                            const double* init, PfSmem<N>& sm, const AMap<N>* inc,
                            const double* agg_pub) {
    const int t = threadIdx.x;
    if (GRID && ch.c > 0) {
        AMap<N> pm;
        pf_carry<N>(agg_pub, ch.c, sm, pm);
        if (t == 0) {
            double x0[N], x1[N];
#pragma unroll
            for (int i = 0; i < N; ++i) x0[i] = init ? init[i] : 0.0;
            amap_apply(pm, x0, x1);
#pragma unroll
            for (int i = 0; i < N; ++i) sm.xs[i] = x1[i];
        }
    } else if (t == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) sm.xs[i] = init ? init[i] : 0.0;
    }
    __syncthreads();
    double part = 0.0;
    if (t < ch.nact) {
        double x[N], y[N], xs[N];
#pragma unroll
        for (int i = 0; i < N; ++i) xs[i] = sm.xs[i];
        if (t == 0) {
#pragma unroll
            for (int i = 0; i < N; ++i) x[i] = xs[i];
        } else {
            const AMap<N> pm = inc[t - 1];
            amap_apply(pm, xs, x);
        }
        const int pa = ch.p0 + t * ch.L, pb = min(pa + ch.L, ch.p0 + ch.cnt);
        AMap<N> m;
        for (int p = pa; p < pb; ++p) {
            const int k = FWD ? p : T - 1 - p;
            mapf(k, m);
            amap_apply(m, x, y);
            part += out(k, x, y);
#pragma unroll
            for (int i = 0; i < N; ++i) x[i] = y[i];
        }
    }
    return part;
}

// Block sum in a fixed order (valid in thread 0).
__device__ __forceinline__ double pf_block_sum(double v, double* red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < RS_WARPS; ++w) s += red[w];
    __syncthreads();
    return s;
}

template <int N, int M>
struct PlanFusedArgs {
    int T, d, it0, maxit;
    double dt, eta;
    const double* s0;
    const double* prm;
    const double* P;      // (d, N)
    const double* Q;
    const double* R;
    const double* clamp;  // nullable
    // stored Riccati phase (element-major, plan_update mode 0)
    const double* K;
    const double* Lg;
    const double* Acl;
    const double* Gm;
    double* dff;          // (T, M)
    double* U0;           // controls of even iterations
    double* U1;           // odd
    double* S0;           // states of even iterations
    double* S1;
    double* lqr_costs;
    unsigned long long* phase_ns;  // [3]: rollout, flow, LQR device time
    int const_off;        // bytes into dynamic smem of the Riccati-array copy (0: none)
    // grid scratch
    double* agg;          // PF_CARRY maps
    double* part;         // PF_CARRY
    int* ipart;           // PF_CARRY
};

__device__ __forceinline__ unsigned long long pf_clock() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// CTA-uniform read of a grid-group value
__device__ __forceinline__ int pf_min_over(const int* v, int n, int* ired) {
    int m = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += RS_BLOCK) m = min(m, __ldcg(v + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) ired[threadIdx.x >> 5] = m;
    __syncthreads();
    int r = 0x7fffffff;
    for (int w = 0; w < RS_WARPS; ++w) r = min(r, ired[w]);
    __syncthreads();
    return r;
}

template <int D, bool GRID, class Mdl>
__global__ void __launch_bounds__(RS_BLOCK, 1)
    rs_plan_kernel(RsArgs A0, PlanFusedArgs<Mdl::N, Mdl::M> pf) {
    constexpr int N = Mdl::N, M = Mdl::M;
    __shared__ double s_pg[N * N + N * M];
    __shared__ int s_first_bad, s_fail, s_stop;
    PfSmem<N>& sm = *reinterpret_cast<PfSmem<N>*>(rs_smem);
    const int tid = threadIdx.x;
    const int b = GRID ? 0 : (int)blockIdx.x;  // problem
    const RsGroup<GRID> grp{GRID ? (int)blockIdx.x : 0, GRID ? (int)gridDim.x : 1, A0.bar};
    const int T = pf.T;
    int* plan_state = A0.plan_state + 8 * b;
    if (GRID) rs_start_epoch(A0);
    if (*((volatile const int*)plan_state) != 0) return;  // uniform: set before the launch
    if (tid == 0) phigam_compute<Mdl>(pf.prm + 0, pf.dt, s_pg);
    // per-problem views (batched: problem b)
    const size_t oTM = (size_t)b * T * M, oTN = (size_t)(b) * (T + 1) * N, oTd = (size_t)b * T * D;
    const double* s0 = pf.s0 + (size_t)b * N;
    double* dff = pf.dff + oTM;
    double* flow = A0.flow + oTd;
    double* X = const_cast<double*>(A0.X) + oTd;
    double* lqr_costs = pf.lqr_costs + (size_t)b * pf.maxit;
    const LiftedFlow<N> lift{flow, pf.P, pf.d};
    // target moments: fixed for the launch (the flows reuse them)
    __shared__ double s_ystat[4];
    {
        __shared__ double s_red8[RS_WARPS][8];
        rs_block_moments<D>(A0.Y + (size_t)b * A0.m * D, A0.m, s_red8, s_ystat);
    }
    bool first = true;
    bool pending_finish = false;
    int pending_it = 0;
    const PfChunk chF = pf_chunk<true, GRID>(T, grp);
    const PfChunk chB = pf_chunk<false, GRID>(T, grp);
    unsigned long long tr = 0, tf = 0, tl = 0;
    // Riccati arrays of this CTA's steps, copied once into shared memory
    // (grid groups, few steps per CTA): the scans then build their maps
    // without L2 round trips.  Same element-major layout with the chunk
    // length as stride; the pointers are offset by -k0 so that the functors'
    // (element * stride + k) indexing is unchanged.
    const double* rAcl = pf.Acl;
    const double* rK = pf.K;
    const double* rLg = pf.Lg;
    const double* rGm = pf.Gm;
    int rstride = T;
    if (GRID && pf.const_off > 0) {
        double* cs = reinterpret_cast<double*>(reinterpret_cast<char*>(rs_smem) + pf.const_off);
        const int cnt = chF.cnt;
        double* sAcl = cs;
        double* sK = sAcl + (size_t)N * N * cnt;
        double* sLg = sK + (size_t)M * N * cnt;
        double* sGm = sLg + (size_t)M * N * cnt;
        for (int i = tid; i < N * N * cnt; i += RS_BLOCK) {
            const int e = i / cnt, k = i - e * cnt;
            sAcl[i] = __ldg(pf.Acl + (size_t)e * T + chF.k0 + k);
        }
        for (int i = tid; i < M * N * cnt; i += RS_BLOCK) {
            const int e = i / cnt, k = i - e * cnt;
            sK[i] = __ldg(pf.K + (size_t)e * T + chF.k0 + k);
            sLg[i] = __ldg(pf.Lg + (size_t)e * T + chF.k0 + k);
            sGm[i] = __ldg(pf.Gm + (size_t)e * T + chF.k0 + k);
        }
        rAcl = sAcl - chF.k0;
        rK = sK - chF.k0;
        rLg = sLg - chF.k0;
        rGm = sGm - chF.k0;
        rstride = cnt;
    }
    __syncthreads();
    for (int it = pf.it0; it < pf.maxit; ++it) {
        double* U = ((it & 1) ? pf.U1 : pf.U0) + oTM;
        double* Un = ((it & 1) ? pf.U0 : pf.U1) + oTM;
        double* S = ((it & 1) ? pf.S1 : pf.S0) + oTN;
        const unsigned long long t0 = pf_clock();
        RS_MARK(50);
        // ---- rollout of U (dynamics.py:276-312) -> S, X -------------------
        if (tid == 0) s_first_bad = 0x7f7f7f7f;
        {
            const RollMap<N, M> mapf{s_pg, U};
            const AMap<N>* inc = pf_phase1<N, true>(T, chF, mapf, sm, GRID ? pf.agg : nullptr);
            if (GRID && first) rs_wait_epoch(A0);
            first = false;
            RS_MARK(51);
            grp.sync();
            RS_MARK(52);
            if (pending_finish && (!GRID || grp.rank == 0) && tid < 32) {
                // the previous update's total cost (fixed order over CTAs)
                const double tot = rs_ordered_sum(pf.part, grp.size);
                int f = -1;
                if (tid == 0) lqr_finish_body(tot, &f, nullptr, lqr_costs, plan_state, pending_it);
            }
            pending_finish = false;
            const RollOut<Mdl> out{S, s0, X, pf.P, pf.d, &s_first_bad, pf.prm, U, pf.dt};
            pf_phase2<N, true, GRID>(T, chF, mapf, out, s0, sm, inc, GRID ? pf.agg : nullptr);
            __syncthreads();
            if (GRID && tid == 0) pf.ipart[grp.rank] = s_first_bad;
            RS_MARK(53);
            grp.sync();
            RS_MARK(54);
            const int fb = GRID ? pf_min_over(pf.ipart, grp.size, sm.ired) : s_first_bad;
            if (fb < 0x7f7f7f7f) {
                if ((!GRID || grp.rank == 0) && tid == 0) roll_finish_body(fb, nullptr, plan_state, it);
                break;
            }
        }
        const unsigned long long t1 = pf_clock();
        RS_MARK(55);
        // ---- flow ------------------------------------------------------------
        {
            RsArgs A = A0;
            A.iteration = it;
            A.ystat = s_ystat;
            rs_flow_body<D, GRID>(A, false);
        }
        const unsigned long long t2 = pf_clock();
        RS_MARK(56);
        // ---- LQR affine phase (lqr.py:180-200 on the stored Riccati phase) ---
        if (tid == 0) {
            s_fail = -1;
        }
        const EtaMap<N, LiftedFlow<N>> emap{rAcl, pf.Q, pf.dt, rstride, lift};
        const AMap<N>* incE = pf_phase1<N, false>(T, chB, emap, sm, GRID ? pf.agg : nullptr);
        RS_MARK(57);
        grp.sync();  // flow statistics and stop flags visible
        RS_MARK(58);
        if (tid == 0) s_stop = *((volatile const int*)plan_state);
        __syncthreads();
        if (s_stop != 0) break;
        {
            const EtaOut<N, M> eout{rLg, dff, &s_fail, rstride};
            pf_phase2<N, false, GRID>(T, chB, emap, eout, nullptr, sm, incE, GRID ? pf.agg : nullptr);
        }
        __syncthreads();
        if (GRID && tid == 0) pf.ipart[grp.rank] = -s_fail;  // min of -fail = -max fail
        const ZMap<N, M> zmap{rAcl, rGm, dff, rstride};
        const AMap<N>* incZ = pf_phase1<N, true>(T, chF, zmap, sm, GRID ? pf.agg + (size_t)PF_CARRY * (N * N + N) : nullptr);
        RS_MARK(59);
        grp.sync();
        RS_MARK(60);
        const int fail_all = GRID ? -pf_min_over(pf.ipart, grp.size, sm.ired) : s_fail;
        if (fail_all >= 0) {
            if ((!GRID || grp.rank == 0) && tid == 0) {
                int f = fail_all;
                lqr_finish_body(0.0, &f, nullptr, lqr_costs, plan_state, it);
            }
            break;
        }
        if (tid == 0) s_fail = -1;
        __syncthreads();
        const ZOut<N, M, LiftedFlow<N>> zout{rK, rstride, dff, pf.Q, pf.R, pf.dt, lift, &s_fail,
                                              nullptr, nullptr, U, Un, pf.eta, pf.clamp};
        const double c = pf_phase2<N, true, GRID>(T, chF, zmap, zout, nullptr, sm, incZ,
                                                  GRID ? pf.agg + (size_t)PF_CARRY * (N * N + N) : nullptr);
        const double cs = pf_block_sum(c, sm.red);
        if (GRID) {
            if (tid == 0) pf.part[grp.rank] = cs;
            pending_finish = true;
            pending_it = it;
        } else if (tid == 0) {
            int f = -1;
            lqr_finish_body(cs, &f, nullptr, lqr_costs, plan_state, it);
        }
        const unsigned long long t3 = pf_clock();
        RS_MARK(61);
        tr += t1 - t0;
        tf += t2 - t1;
        tl += t3 - t2;
        __syncthreads();
    }
    if (GRID && pending_finish) {
        grp.sync();
        if (grp.rank == 0 && tid < 32) {
            const double tot = rs_ordered_sum(pf.part, grp.size);
            int f = -1;
            if (tid == 0) lqr_finish_body(tot, &f, nullptr, lqr_costs, plan_state, pending_it);
        }
    }
    if (tid == 0 && (!GRID || grp.rank == 0) && pf.phase_ns) {
        unsigned long long* pn = pf.phase_ns + 3 * b;
        pn[0] += tr;
        pn[1] += tf;
        pn[2] += tl;
    }
}

}  // namespace fcb
