// plan_stein.cuh -- the SVGD coverage loop of a linear model in ONE persistent
// launch (optimizer.py:221-269 with the flow of stein.py:66-122), the Stein
// counterpart of rs_plan_kernel (plan_fused.cuh).  Per iteration, one CTA per
// SM, grid barriers between the phases:
//
//   rollout   affine scan of s_{k+1} = Phi s_k + Gam u_k -> S, X = P S[1:]
//             (plan_fused.cuh's pf_phase1/2, CTA r owns steps [T r/G, T (r+1)/G))
//   score     GaussianMixture score of the CTA's own points (reference.py:103-110)
//   bandwidth exact median of all T^2 distances by radix passes over the
//             grid: every CTA histograms its run of the T (T-1) / 2 pairs in
//             shared memory, adds the nonzero bins into a rotating global
//             histogram, and after the barrier every CTA selects the digit
//             from the global counts itself (identical inputs, identical
//             prefixes: no broadcast barrier); once the selected bucket holds
//             <= SVP_CAND keys (after two passes at config 1) they are
//             gathered and ranked exactly; h = med^2 / log(T+1)
//   flow      g_i = (1/T)[sum_j k_ij s_j + (2/h)(x_i sum_j k_ij - sum_j k_ij x_j)]
//             for the CTA's own rows against all T points in shared memory
//             (fp64, the per-iteration path's centred / scaled form)
//   LQR       eta / z scans on the stored Riccati phase, U <- clamp(U + eta v*)
//
// The flow rows a CTA computes are the LQR steps it owns, so flow -> LQR is
// CTA-local; the mean flow magnitude (the convergence statistic) is summed in
// CTA order after the LQR's first barrier, by every CTA.  Included at the end
// of dynamics.cu after plan_fused.cuh.
#pragma once

#include "plan_fused.cuh"
#include "stein_dev.cuh"

namespace fcb {

constexpr int SVP_BINS = 2048;
constexpr int SVP_CAND = 1024;  // candidate cap of the final O(m^2) rank select

template <int N, int M>
struct SvFusedArgs {
    PlanFusedArgs<N, M> pf;
    double* X;            // (T, D) projected rollout states: the flow's points
    double* flow;         // (T, D)
    double* scores;       // (T, D)
    const double* gmm;    // mixture parameters (gmm_point layout)
    int k;                // mixture components
    double bw_fixed;      // > 0: fixed bandwidth (no median)
    double log_np1;
    double conv_tol;
    double* fstat;        // [8], as stein_finalize_kernel
    int* plan_state;      // [8]
    double* flow_log;     // [4 * maxit]
    unsigned* hist;       // 3 x 2 x SVP_BINS rotating radix histograms (first two zeroed)
    unsigned long long* cand;  // SVP_CAND keys gathered for the final select
    unsigned* ccount;     // 2 rotating candidate counters (zeroed)
    double* npart;        // per-CTA sums of |g_i|
    GridBarrier* bar;
    unsigned* done;
    unsigned launch_id;
    int sv_off;           // bytes into dynamic smem of the flow's column set
};

struct SvpSel {
    unsigned long long pre[2], rank[2];
    unsigned long long warp[2][RS_WARPS];
    unsigned long long wbase[2][RS_WARPS];
    unsigned long long nw[2][3];
    unsigned long long bcnt[2];  // count of the selected bin (pairs x2, zeros included)
};

// Digit selection from the global counts of one pass (every CTA, RS_BLOCK
// threads); the n diagonal zeros sit in bin 0 while the prefix is 0.
__device__ void svp_select(const unsigned* g, int n, int pass, SvpSel& s) {
    constexpr int PER = SVP_BINS / RS_BLOCK;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int bits = med_pass_bits(pass), nbins = 1 << bits;
    const unsigned long long p0 = s.pre[0], p1 = s.pre[1];
    const bool same = p0 == p1;
    unsigned long long c[2][PER], sum[2], incl[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const unsigned* h = g + (same ? 0 : t) * SVP_BINS;
        const unsigned long long z = ((t ? p1 : p0) == 0ull) ? (unsigned long long)n : 0ull;
        sum[t] = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int b = tid * PER + k;
            c[t][k] = (b < nbins) ? (unsigned long long)__ldcg(h + b) + (b == 0 ? z : 0ull) : 0ull;
            sum[t] += c[t][k];
        }
        incl[t] = sum[t];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long v = __shfl_up_sync(0xffffffffu, incl[t], o);
            if (lane >= o) incl[t] += v;
        }
        if (lane == 31) s.warp[t][wid] = incl[t];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const unsigned long long w = lane < RS_WARPS ? s.warp[t][lane] : 0ull;
            unsigned long long x = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long v = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += v;
            }
            if (lane < RS_WARPS) s.wbase[t][lane] = x - w;
        }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const unsigned long long excl = s.wbase[t][wid] + incl[t] - sum[t];
        const unsigned long long r = s.rank[t];
        const bool last = tid == RS_BLOCK - 1;
        if ((r >= excl && r < excl + sum[t]) || (last && r >= excl + sum[t])) {
            unsigned long long rr = r - excl;
            int b = tid * PER;
            unsigned long long cb = 0;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                cb = c[t][k];
                if (rr < c[t][k] || k == PER - 1) break;
                rr -= c[t][k];
                ++b;
            }
            b = min(b, nbins - 1);
            s.nw[t][0] = ((t ? p1 : p0) << bits) | (unsigned long long)b;
            s.nw[t][1] = rr;
            s.nw[t][2] = cb;
        }
    }
    __syncthreads();
    if (tid == 0) {
        s.pre[0] = s.nw[0][0];
        s.rank[0] = s.nw[0][1];
        s.bcnt[0] = s.nw[0][2];
        s.pre[1] = s.nw[1][0];
        s.rank[1] = s.nw[1][1];
        s.bcnt[1] = s.nw[1][2];
    }
    __syncthreads();
}

// Exact select among the gathered candidates (every CTA): bucket t's multiset
// is z zeros (the diagonal, while its prefix is 0) and every candidate twice.
__device__ void svp_resolve(const unsigned long long* cand, int m, int kshift, int n,
                            SvpSel& s) {
    __shared__ unsigned long long s_res[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const unsigned long long pre = s.pre[t];
        const unsigned long long z = (pre == 0ull) ? (unsigned long long)n : 0ull;
        const unsigned long long rr = s.rank[t];
        if (threadIdx.x == 0 && rr < z) s_res[t] = 0ull;
        if (rr >= z) {
            const unsigned long long r = rr - z;
            for (int i = threadIdx.x; i < m; i += RS_BLOCK) {
                const unsigned long long c = cand[i];
                if ((c >> kshift) != pre) continue;
                unsigned long long less = 0, eq = 0;
                for (int j = 0; j < m; ++j) {
                    const unsigned long long x = cand[j];
                    if ((x >> kshift) != pre) continue;
                    less += x < c;
                    eq += x == c;
                }
                if (2ull * less <= r && r < 2ull * (less + eq)) s_res[t] = c;  // equal writers
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s.pre[0] = s_res[0];
        s.pre[1] = s_res[1];
    }
    __syncthreads();
}

// pair q of the row-major upper triangle (i < j), folded into an H x W
// rectangle (rectangle row r: triangle row r, then its partner row)
__device__ __forceinline__ void svp_pair(int n, long long q, int& i, int& j) {
    const bool even = (n & 1) == 0;
    const long long W = even ? n - 1 : n;
    const int r = (int)(q / W);
    const int c = (int)(q - (long long)r * W);
    const int len = n - 1 - r;
    if (c < len) {
        i = r;
        j = r + 1 + c;
    } else {
        i = even ? n - 1 - r : n - 2 - r;
        j = i + 1 + (c - len);
    }
}

// The exact median bandwidth over the grid (stein.py:66-76); hstat -> s_h
// in every CTA.  gpass counts the launch's radix passes (buffer rotation).
template <int D>
__device__ void svp_median(const double* __restrict__ X, int n, double log_np1, unsigned* ghist,
                           unsigned long long* gcand, unsigned* gcount, unsigned& ggather,
                           const RsGroup<true>& grp, unsigned& gpass, unsigned* shist,
                           SvpSel& sel, double* s_h) {
    const int tid = threadIdx.x;
    const unsigned long long NN = (unsigned long long)n * (unsigned long long)n;
    if (tid == 0) {
        sel.pre[0] = sel.pre[1] = 0ull;
        sel.rank[0] = (NN - 1ull) / 2ull;
        sel.rank[1] = NN / 2ull;
    }
    const long long P = (long long)n * (n - 1) / 2;
    const long long q0 = P * grp.rank / grp.size, q1 = P * (grp.rank + 1) / grp.size;
    for (int pass = 0; pass < 6; ++pass) {
        const int shift = med_pass_shift(pass), bits = med_pass_bits(pass);
        const int hshift = shift + bits;
        for (int b = tid; b < 2 * SVP_BINS; b += RS_BLOCK) shist[b] = 0u;
        __syncthreads();
        const unsigned long long pre0 = sel.pre[0], pre1 = sel.pre[1];
        const bool same = pre0 == pre1;
        for (long long q = q0 + tid; q < q1; q += RS_BLOCK) {
            int i, j;
            svp_pair(n, q, i, j);
            // other CTAs wrote X this iteration: read through L2, not a stale L1 line
            double xi[D], xj[D];
#pragma unroll
            for (int c = 0; c < D; ++c) {
                xi[c] = __ldcg(X + (size_t)i * D + c);
                xj[c] = __ldcg(X + (size_t)j * D + c);
            }
            const unsigned long long key = sqdist_key<D>(xi, xj);
            const unsigned long long hi = (hshift >= 64) ? 0ull : (key >> hshift);
            const unsigned dig = (unsigned)((key >> shift) & ((1ull << bits) - 1ull));
            if (hi == pre0) atomicAdd(&shist[dig], 2u);
            if (!same && hi == pre1) atomicAdd(&shist[SVP_BINS + dig], 2u);
        }
        __syncthreads();
        unsigned* g = ghist + (size_t)(gpass % 3u) * 2 * SVP_BINS;
        for (int b = tid; b < 2 * SVP_BINS; b += RS_BLOCK)
            if (shist[b]) atomicAdd(&g[b], shist[b]);
        grp.sync();
        // the buffer of pass gpass + 2 was last read before this barrier
        if (grp.rank == 0) {
            unsigned* z = ghist + (size_t)((gpass + 2u) % 3u) * 2 * SVP_BINS;
            for (int b = tid; b < 2 * SVP_BINS; b += RS_BLOCK) z[b] = 0u;
        }
        svp_select(g, n, pass, sel);
        ++gpass;
        // few keys left in the selected bucket(s): gather them and rank them
        // exactly instead of running the remaining passes (one barrier for four)
        if (pass + 1 < 6) {
            unsigned long long m = 0;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                if (t == 1 && sel.pre[1] == sel.pre[0]) break;
                const unsigned long long z = (sel.pre[t] == 0ull) ? (unsigned long long)n : 0ull;
                m += (sel.bcnt[t] - min(z, sel.bcnt[t])) / 2ull;
            }
            if (m <= (unsigned long long)SVP_CAND) {  // grid-uniform
                unsigned* cnt = gcount + (ggather & 1u);
                const unsigned long long k0 = sel.pre[0], k1 = sel.pre[1];
                for (long long q = q0 + tid; q < q1; q += RS_BLOCK) {
                    int i, j;
                    svp_pair(n, q, i, j);
                    double xi[D], xj[D];
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        xi[c] = __ldcg(X + (size_t)i * D + c);
                        xj[c] = __ldcg(X + (size_t)j * D + c);
                    }
                    const unsigned long long key = sqdist_key<D>(xi, xj);
                    const unsigned long long hi = key >> shift;
                    if (hi == k0 || hi == k1) {
                        const unsigned slot = atomicAdd(cnt, 1u);
                        if (slot < (unsigned)SVP_CAND) gcand[slot] = key;
                    }
                }
                grp.sync();
                // the other counter is next used by the next gather (next iteration)
                if (grp.rank == 0 && tid == 0) gcount[(ggather + 1u) & 1u] = 0u;
                ++ggather;
                const int mm = (int)min(__ldcg(cnt), (unsigned)SVP_CAND);
                unsigned long long* sc = reinterpret_cast<unsigned long long*>(shist);
                for (int c = tid; c < mm; c += RS_BLOCK) sc[c] = __ldcg(gcand + c);
                __syncthreads();
                svp_resolve(sc, mm, shift, n, sel);
                break;
            }
        }
    }
    if (tid == 0) median_finish_vals(sel.pre[0], sel.pre[1], n, log_np1, s_h);
    __syncthreads();
}

// The flow phase of one iteration over the grid (every CTA): scores of the
// CTA's points [k0, k1), the bandwidth (exact median or fixed), the Stein flow
// of those rows and the CTA's sum of |g_i| in npart.  The rows become visible
// grid-wide at the caller's next barrier.
template <int D, class Args>
__device__ void svp_flow_phase(const Args& a, int T, int k0, int k1, const RsGroup<true>& grp,
                               unsigned& gpass, unsigned& ggather, unsigned* shist, SvpSel& sel,
                               double* s_h, double* s_rownorm, double* cx, double* cw) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const double* X = a.X;
    for (int i = k0 + tid; i < k1; i += RS_BLOCK) {
        double xi[D];
#pragma unroll
        for (int q = 0; q < D; ++q) xi[q] = __ldcg(X + (size_t)i * D + q);
        gmm_point<D>(xi, a.k, a.gmm, a.scores + (size_t)i * D, nullptr);
    }
    if (a.bw_fixed > 0.0) {
        if (tid == 0) {
            const bool clamped = a.bw_fixed <= BANDWIDTH_FLOOR;
            s_h[0] = clamped ? BANDWIDTH_FLOOR : a.bw_fixed;
            s_h[1] = NAN;
            s_h[2] = clamped ? 1.0 : 0.0;
            s_h[3] = 0.0;
        }
        grp.sync();  // scores complete
    } else {
        // the first pass's barrier also publishes the scores
        svp_median<D>(X, T, a.log_np1, a.hist, a.cand, a.ccount, ggather, grp, gpass, shist, sel,
                      s_h);
    }
    // every point as a column, centred on X[0] and scaled by 1/sqrt(h)
    // (stein_run's form; coincident clouds give x' == 0 exactly)
    const double h = s_h[0];
    const double sc = sqrt(1.0 / h), two_h = 2.0 / h;
    double x0[D];
#pragma unroll
    for (int q = 0; q < D; ++q) x0[q] = __ldcg(X + q);
    for (int e = tid; e < T * D; e += RS_BLOCK) {
        const int q = e % D;
        const double xc = __ldcg(X + e) - x0[q];
        cx[e] = xc * sc;
        cw[e] = __ldcg(a.scores + e) - two_h * xc;
    }
    __syncthreads();
    const double inv_n = 1.0 / T;
    for (int i = k0 + wid; i < k1; i += RS_WARPS) {
        double xi[D], K = 0.0, A[D];
#pragma unroll
        for (int q = 0; q < D; ++q) {
            xi[q] = cx[(size_t)i * D + q];
            A[q] = 0.0;
        }
        for (int j = lane; j < T; j += 32) {
            double d2 = 0.0;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double df = xi[q] - cx[(size_t)j * D + q];
                d2 = fma(df, df, d2);
            }
            const double kk = exp(-d2);
            K += kk;
#pragma unroll
            for (int q = 0; q < D; ++q) A[q] = fma(kk, cw[(size_t)j * D + q], A[q]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            K += __shfl_xor_sync(0xffffffffu, K, o);
#pragma unroll
            for (int q = 0; q < D; ++q) A[q] += __shfl_xor_sync(0xffffffffu, A[q], o);
        }
        if (lane == 0) {
            double sq = 0.0;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double xc = __ldcg(X + (size_t)i * D + q) - x0[q];
                const double g = inv_n * (A[q] + two_h * xc * K);
                a.flow[(size_t)i * D + q] = g;
                sq += g * g;
            }
            s_rownorm[(i - k0) & 63] = sqrt(sq);
        }
    }
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;  // rows in order (at most 64 per CTA, checked on the host)
        for (int i = k0; i < k1; ++i) s += s_rownorm[(i - k0) & 63];
        a.npart[grp.rank] = s;
    }
}

// After the flow norms are visible: the mean |g| (summed in CTA order by every
// CTA, so the stop decision is grid-uniform); CTA 0 writes the statistics and
// planner hooks of stein_finalize_kernel.  Returns the mean.
template <class Args>
__device__ double svp_finish_flow(const Args& a, int T, int it, const RsGroup<true>& grp,
                                  const double* s_h, double* s_mean) {
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int r = 0; r < grp.size; ++r) s += __ldcg(a.npart + r);
        *s_mean = s / T;
        if (grp.rank == 0) {
            const double mm = *s_mean;
            a.fstat[0] = 0.0;
            a.fstat[1] = 1.0;
            a.fstat[2] = 0.0;
            a.fstat[3] = mm;
            a.fstat[4] = s_h[0];
            a.fstat[5] = s_h[2];
            a.fstat[6] = s_h[1];
            a.fstat[7] = 0.0;
            double* lg = a.flow_log + 4 * (size_t)it;
            lg[0] = mm;
            lg[1] = s_h[0];
            lg[2] = s_h[2];
            lg[3] = s_h[1];
            a.plan_state[FCB_STATE_FLOWS] = it + 1;
            if (mm < a.conv_tol) a.plan_state[FCB_STATE_STOP] = 1;
        }
    }
    __syncthreads();
    return *s_mean;
}

// Scans spread over the grid as in rs_plan_kernel: CTA r owns steps
// [T r/G, T (r+1)/G).  (Measured alternative: CTA 0 scanning all T = 500
// steps of config 1 alone while the others wait -- 40 vs 25 us of LQR per
// iteration; the block-wide Hillis-Steele over 128 runs is slower than the
// grid carry.)
template <int D, class Mdl>
__global__ void __launch_bounds__(RS_BLOCK, 1) sv_plan_kernel(SvFusedArgs<Mdl::N, Mdl::M> a) {
    constexpr int N = Mdl::N, M = Mdl::M;
    const PlanFusedArgs<N, M>& pf = a.pf;
    __shared__ double s_pg[N * N + N * M];
    __shared__ int s_first_bad, s_fail;
    __shared__ double s_h[4];
    __shared__ double s_rownorm[64];
    __shared__ double s_mean;
    __shared__ unsigned shist[2 * SVP_BINS];
    __shared__ SvpSel sel;
    PfSmem<N>& sm = *reinterpret_cast<PfSmem<N>*>(rs_smem);
    const int tid = threadIdx.x;
    RsArgs ep{};
    ep.bar = a.bar;
    ep.done = a.done;
    ep.launch_id = a.launch_id;
    rs_start_epoch(ep);
    const RsGroup<true> grp{(int)blockIdx.x, (int)gridDim.x, a.bar};
    const int T = pf.T;
    int* plan_state = a.plan_state;
    if (*((volatile const int*)plan_state) != 0) return;  // uniform: set before the launch
    if (tid == 0) phigam_compute<Mdl>(pf.prm + 0, pf.dt, s_pg);
    double* dff = pf.dff;
    double* X = a.X;
    unsigned gpass = 0, ggather = 0;
    const PfChunk chF = pf_chunk<true, true>(T, grp);  // this CTA's points / steps
    double* cx = reinterpret_cast<double*>(reinterpret_cast<char*>(rs_smem) + a.sv_off);
    double* cw = cx + (size_t)T * D;
    unsigned long long tr = 0, tf = 0, tl = 0;
    const LiftedFlow<N> lift{a.flow, pf.P, pf.d};
    bool first = true;
    bool pending_finish = false;
    int pending_it = 0;
    const PfChunk chB = pf_chunk<false, true>(T, grp);
    // this CTA's Riccati arrays in shared memory (as rs_plan_kernel)
    const double* rAcl = pf.Acl;
    const double* rK = pf.K;
    const double* rLg = pf.Lg;
    const double* rGm = pf.Gm;
    int rstride = T;
    if (pf.const_off > 0) {
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
        double* U = ((it & 1) ? pf.U1 : pf.U0);
        double* Un = ((it & 1) ? pf.U0 : pf.U1);
        double* S = ((it & 1) ? pf.S1 : pf.S0);
        const unsigned long long t0 = pf_clock();
        // ---- rollout of U (dynamics.py:276-312) -> S, X ---------------
        if (tid == 0) s_first_bad = 0x7f7f7f7f;
        {
            const RollMap<N, M> mapf{s_pg, U};
            const AMap<N>* inc = pf_phase1<N, true>(T, chF, mapf, sm, pf.agg);
            if (first) rs_wait_epoch(ep);
            first = false;
            grp.sync();
            if (pending_finish && grp.rank == 0 && tid < 32) {
                const double tot = rs_ordered_sum(pf.part, grp.size);
                int f = -1;
                if (tid == 0) lqr_finish_body(tot, &f, nullptr, pf.lqr_costs, plan_state, pending_it);
            }
            pending_finish = false;
            const RollOut<Mdl> out{S, pf.s0, X, pf.P, pf.d, &s_first_bad, pf.prm, U, pf.dt};
            pf_phase2<N, true, true>(T, chF, mapf, out, pf.s0, sm, inc, pf.agg);
            __syncthreads();
            if (tid == 0) pf.ipart[grp.rank] = s_first_bad;
            grp.sync();  // X complete
            const int fb = pf_min_over(pf.ipart, grp.size, sm.ired);
            if (fb < 0x7f7f7f7f) {
                if (grp.rank == 0 && tid == 0) roll_finish_body(fb, nullptr, plan_state, it);
                break;
            }
        }
        const unsigned long long t1 = pf_clock();
        // ---- Stein flow (stein.py:79-122) -----------------------------
        svp_flow_phase<D>(a, T, chF.k0, chF.k1, grp, gpass, ggather, shist, sel, s_h,
                          s_rownorm, cx, cw);
        const unsigned long long t2 = pf_clock();
        // ---- LQR affine phase (lqr.py:180-200 on the stored Riccati phase)
        if (tid == 0) s_fail = -1;
        const EtaMap<N, LiftedFlow<N>> emap{rAcl, pf.Q, pf.dt, rstride, lift};
        const AMap<N>* incE = pf_phase1<N, false>(T, chB, emap, sm, pf.agg);
        grp.sync();  // flow norms visible
        if (svp_finish_flow(a, T, it, grp, s_h, &s_mean) < a.conv_tol) break;
        {
            const EtaOut<N, M> eout{rLg, dff, &s_fail, rstride};
            pf_phase2<N, false, true>(T, chB, emap, eout, nullptr, sm, incE, pf.agg);
        }
        __syncthreads();
        if (tid == 0) pf.ipart[grp.rank] = -s_fail;
        const ZMap<N, M> zmap{rAcl, rGm, dff, rstride};
        const AMap<N>* incZ =
            pf_phase1<N, true>(T, chF, zmap, sm, pf.agg + (size_t)PF_CARRY * (N * N + N));
        grp.sync();
        const int fail_all = -pf_min_over(pf.ipart, grp.size, sm.ired);
        if (fail_all >= 0) {
            if (grp.rank == 0 && tid == 0) {
                int f = fail_all;
                lqr_finish_body(0.0, &f, nullptr, pf.lqr_costs, plan_state, it);
            }
            break;
        }
        if (tid == 0) s_fail = -1;
        __syncthreads();
        const ZOut<N, M, LiftedFlow<N>> zout{rK, rstride, dff, pf.Q, pf.R, pf.dt, lift, &s_fail,
                                              nullptr, nullptr, U, Un, pf.eta, pf.clamp};
        const double c = pf_phase2<N, true, true>(T, chF, zmap, zout, nullptr, sm, incZ,
                                                  pf.agg + (size_t)PF_CARRY * (N * N + N));
        const double cs = pf_block_sum(c, sm.red);
        if (tid == 0) pf.part[grp.rank] = cs;
        pending_finish = true;
        pending_it = it;
        const unsigned long long t3 = pf_clock();
        tr += t1 - t0;
        tf += t2 - t1;
        tl += t3 - t2;
        __syncthreads();
    }
    if (pending_finish) {
        grp.sync();
        if (grp.rank == 0 && tid < 32) {
            const double tot = rs_ordered_sum(pf.part, grp.size);
            int f = -1;
            if (tid == 0) lqr_finish_body(tot, &f, nullptr, pf.lqr_costs, plan_state, pending_it);
        }
    }
    if (tid == 0 && grp.rank == 0 && pf.phase_ns) {
        pf.phase_ns[0] += tr;
        pf.phase_ns[1] += tf;
        pf.phase_ns[2] += tl;
    }
}

}  // namespace fcb
