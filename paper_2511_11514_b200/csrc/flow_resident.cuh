// flow_resident.cuh -- device side and launch planning of the shared-memory
// resident Sinkhorn flow (flow_resident.cu); also used by the fused planner
// kernel (plan_fused.cuh).
#pragma once
// flow_resident.cu -- sinkhorn_flow with every column set resident in shared
// memory (sinkhorn.py:338-400: resolve_omega :136-148, _lse_rows :151-167,
// _solve_asymmetric :170-205, _solve_symmetric :208-236, gradient :383-391).
//
// For point sets that fit on chip (n + max(n, m) columns, 12-16 B each) the
// chunked solver of sinkhorn.cu pays for its generality with partial buffers
// and merge phases between the sweeps.  Here each CTA of the group keeps a
// full copy of the column records (packed fp32 coordinates 2 s x', and the
// folded potential W = s pot + rowc) in shared memory and OWNS a slice of the
// rows of every sweep, so a row's log-sum-exp is finished inside one CTA:
//
//   setup    every CTA computes the point statistics (same fixed order, so
//            identical omega and centrings everywhere), packs the columns
//   loop     sweep A   rows = own slice of Y, columns X  -> g, publish W_Y
//            sync; reload W_Y
//            sweep B   rows = own slice of X, columns Y  -> f_new, delta,
//                      err, row sums, barycentres; publish W_X
//            sync; err test (grid-uniform); reload W_X
//   self     the same with rows = own X slice, columns X (centred on mean X)
//   end      envelope gradient for the own rows; the last CTA to finish
//            writes the statistics, warm-state flags and planner hooks.
//
// A "group" is the whole grid (one problem, grid barrier between sweeps) or a
// single CTA (batched independent problems, one per CTA; the exchange is
// shared memory and the sync is __syncthreads).
//
// Pair arithmetic (log2 units, expanded form as in sinkhorn.cu): for row i and
// column j, t = W_j + x'_i . Yh_j + rc_i with rc_i = rowc_i - shift_i, the
// shift being the row's LSE estimate from its own current potential (exact at
// the fixed point).  Columns are processed in quads with packed FFMA2/FADD2
// (two columns per instruction, the row value as a scalar operand); one
// MUFU.EX2 per pair.  An 8-column sub-tile whose sum leaves [2^-64, 2^64]
// takes the rare re-shift path.  Threads of a row group split the columns;
// their (shift, sum, moments) partials are combined by a symmetric butterfly
// (bit-identical in every lane) and, across warps, in fixed order -- no float
// atomics, results are deterministic.
#include "fcb_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <atomic>

namespace fcb {

constexpr int RS_BLOCK = 512;
constexpr int RS_WARPS = RS_BLOCK / 32;
constexpr int RS_MIN_CG_LOG = 3;  // >= 8 column threads per row group
constexpr double RS_EXP_CLIP = 500.0;       // sinkhorn.py:67
constexpr double RS_OMEGA_FLOOR = 1e-12;    // sinkhorn.py:66
constexpr double RS_AUTO_OMEGA = 0.05;      // sinkhorn.py:65

#ifdef FCB_TIMELINE
__device__ unsigned long long g_rs_tl[16384];
__device__ unsigned g_rs_tl_n;
#define RS_MARK(tag)                                                              \
    do {                                                                          \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                \
            unsigned long long t_;                                                \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));               \
            unsigned i_ = g_rs_tl_n;                                              \
            if (i_ < 16384) g_rs_tl[i_] = (t_ << 8) | (unsigned long long)(tag);  \
            g_rs_tl_n = i_ + 1;                                                   \
        }                                                                         \
    } while (0)
#else
#define RS_MARK(tag) \
    do {             \
    } while (0)
#endif

// rows per thread per pass, at most (register budget at 512 threads)
// (the moment sweeps carry 2D more accumulators per row)
template <int D, bool BARY> struct RsMaxNr { static constexpr int value = BARY ? 4 : 6; };
template <bool BARY> struct RsMaxNr<3, BARY> { static constexpr int value = BARY ? 3 : 4; };

// per-sweep thread layout: 2^cg column threads per row group, nr rows per
// thread per pass
struct RsPlan {
    int cg, nr;
};

// per-problem arguments (batched problems: pointer + b * stride)
struct RsArgs {
    const double* X;   // (n, D) per problem
    const double* Y;   // (m, D)
    int n, m;
    double omega_fixed;
    int max_iters;
    double tol, conv_tol;
    double* warm_f;    // (n) nullable
    double* warm_p;
    int* warm_valid;   // [2]
    double* flow;      // (n, D)
    double* fstat;     // [8]
    int* plan_state;   // [8] nullable
    int iteration;
    double* flow_log;  // [4 * iters] nullable
    long long log_stride;  // flow_log doubles per problem (batched)
    // workspace (per problem)
    double* fbuf;      // 2 n: f ping-pong
    double* pbuf;      // 2 n: p ping-pong
    double* gbuf;      // m
    float* WX;         // grid groups: published folded potentials
    float* WY;
    float* WS;         // self term: 2 published buffers per problem (ldWS floats each)
    int ldWS;
    double* dx;        // n: delta of the last cross update
    double* bx;        // n (D + 1): log plan row mass, barycentre
    double* dp;        // n: the same for the self term
    double* bp;
    unsigned long long* errslot;  // 4 per problem
    double* fin_part;  // group size (grid) or batch
    unsigned* done;    // last-CTA counter
    GridBarrier* bar;
    RsPlan plA, plB, plS;     // thread layouts of the three sweeps
    int nqpA, nqpB, nqpS;     // padded quads of the three column sets
    int ldA, ldB;             // floats per array of smem regions A and B
    int cache_off, cache_rows;  // own-row cache (floats offset, rows; 0: none)
    unsigned launch_id;         // grid groups: epoch of this launch (barrier reset)
    const double* ystat;        // nullable: precomputed target moments [4]
};

// Shared-memory column set: D coordinate arrays and the folded potential,
// structure of arrays (float offsets into rs_smem), quads read with LDS.128.
// Columns are padded with W = -inf to `nqp` quads, a multiple of twice the
// column threads of every sweep that reads the set, so the pair loop has no
// bounds checks.
extern __shared__ __align__(16) float rs_smem[];

struct RsCols {
    int q[3];
    int w;
    int nq;   // live quads (ceil(columns / 4))
    int nqp;  // padded quads
};

struct RsRes {  // combined row partial
    float k, s, a[3];
};



// Barriers passed by this CTA in the current launch (grid groups): the
// arrival target is known locally, so an arrival is a fire-and-forget
// red.release (no atomic round trip) and only the poll waits.
__shared__ unsigned long long rs_bar_gen;
#ifndef RS_BAR_SLEEP
#define RS_BAR_SLEEP 20  // ns between polls of the grid barrier
#endif

template <bool GRID>
struct RsGroup {
    int rank, size;
    GridBarrier* bar;
    __device__ __forceinline__ void sync() const {
        if constexpr (GRID) {
            __syncthreads();
            FCB_TL_MARK();
            if (threadIdx.x == 0) {
                // 64-bit arrival counter: no wrap within a launch
                const unsigned long long target = (rs_bar_gen + 1ull) * (unsigned long long)size;
                rs_bar_gen += 1ull;
                asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&bar->count)
                             : "memory");
                while (ld_acquire_u64(&bar->count) < target) __nanosleep(RS_BAR_SLEEP);
            }
            __syncthreads();
            FCB_TL_MARK();
        } else {
            __syncthreads();
        }
    }
};

// Copy the published folded potentials of a column set into shared memory
// (grid groups; `src` holds nq * 4 floats, padded with -inf).
__device__ __forceinline__ void rs_reload(const RsCols& cs, const float* src) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(rs_smem + cs.w);
#pragma unroll 4
    for (int j = threadIdx.x; j < cs.nq; j += RS_BLOCK) d4[j] = __ldcg(s4 + j);
}

// exp2 of a packed pair on the FMA pipe (offloads the MUFU queue in the pair
// loop): t = j + f with j = rint(t), f in [-1/2, 1/2]; 2^f by a degree-5
// near-minimax polynomial (relative error 3.5e-7 in fp32, MUFU.EX2's is
// ~2.4e-7) and 2^j added into the exponent field.  t is clamped to
// [-127, 127]: 2^-127 comes out as exactly 0 (the -inf padding columns), and
// the exponent never wraps.  Off by default: measured in scripts/micro/
// rs_loop.cu, offloading one pair in four is neutral for the plain sweeps and
// 10-15 points slower for the moment sweeps (the loop is issue-bound there,
// not MUFU-bound).
#ifndef RS_EMU
#define RS_EMU 0
#endif
__device__ __forceinline__ float2 rs_ex2_poly2(float2 t) {
    t.x = fminf(fmaxf(t.x, -127.f), 127.f);
    t.y = fminf(fmaxf(t.y, -127.f), 127.f);
    const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
    const float2 y = __fadd2_rn(t, magic);
    const float2 j = __fadd2_rn(y, make_float2(-12582912.f, -12582912.f));
    const float2 f = __fadd2_rn(t, make_float2(-j.x, -j.y));
    float2 p = make_float2(0.0012915670f, 0.0012915670f);
    p = __ffma2_rn(p, f, make_float2(0.0096685309f, 0.0096685309f));
    p = __ffma2_rn(p, f, make_float2(0.055516887f, 0.055516887f));
    p = __ffma2_rn(p, f, make_float2(0.24022265f, 0.24022265f));
    p = __ffma2_rn(p, f, make_float2(0.69314647f, 0.69314647f));
    p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(y.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(y.y) << 23)));
}

// Rows whose streaming pass was refused and redone by rs_careful (diagnostics
// for the parity tests; one atomic per refused row, off the common path).
// static: every translation unit that instantiates the kernels has its own.
static __device__ unsigned g_rs_careful_rows;

// A row sum is trusted in [2^-64, 2^120]: below, nothing has been
// accumulated under a too-high shift estimate; above (or inf / NaN), the
// terms overflowed.  Positive floats order like their bit patterns, so the
// test is one unsigned compare.
__device__ __forceinline__ bool rs_out_of_range(float s) {
    constexpr unsigned LO = 0x1F800000u;  // 2^-64
    constexpr unsigned HI = 0x7B800000u;  // 2^120
    return (__float_as_uint(s) - LO) > (HI - LO);
}

// ---------------------------------------------------------------------------
// one pass of a sweep: NR rows per thread (rows pb + rg + RG r of the CTA's
// slice) against every column in shared memory
// ---------------------------------------------------------------------------
// Rows: init(li, x[D], rc) for the slice-local row li and rowc2(li) (double,
// log2 units), rc == (float)(rowc2 - shift2).  epi(li, L, bar[D]): the natural
// unit LSE and (BARY) the column moments / sum.
//
// The pair loop is straight-line across the NR rows (no per-row branches, so
// the scheduler interleaves rows): a row's sub-tile sum and moments are
// committed only after one joint range test, and the rare re-shift runs out
// of line for the rows that failed it.
// Eight columns (quads q0, q1) of a shared-memory column set.
template <int D>
__device__ __forceinline__ void rs_load8(const float4* wv, const float4* const* qv, int q0, int q1,
                                         float* w, float (*y)[8]) {
    const float4 w0 = wv[q0], w1 = wv[q1];
    w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
    w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
#pragma unroll
    for (int q = 0; q < D; ++q) {
        const float4 a0 = qv[q][q0], a1 = qv[q][q1];
        y[q][0] = a0.x; y[q][1] = a0.y; y[q][2] = a0.z; y[q][3] = a0.w;
        y[q][4] = a1.x; y[q][5] = a1.y; y[q][6] = a1.z; y[q][7] = a1.w;
    }
}

// Careful pass for one row over this thread's columns (rare): per 8-column
// sub-tile, a sum that would leave [2^-64, 2^64] (or is the first mass under a
// too-high shift) re-shifts the row by the sub-tile max first.
struct RsRowState {
    float x[3];
    float rc, sum;
    float2 acc[3];
};

template <int D, bool BARY>
__device__ __noinline__ RsRowState rs_careful(const float4* wv, const float4* const* qv, int cg,
                                              int cg_log, int steps, RsRowState st) {
    const float BIG = 1.8446744e19f, TINY = 5.421011e-20f;  // 2^64, 2^-64
    st.sum = 0.f;
#pragma unroll
    for (int q = 0; q < D; ++q) st.acc[q] = make_float2(0.f, 0.f);
    for (int kk = 0; kk < steps; kk += 2) {
        const int q0 = cg + (kk << cg_log), q1 = q0 + (1 << cg_log);
        float w[8], y[D][8];
        rs_load8<D>(wv, qv, q0, q1, w, y);
        float t[8], e[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float a = w[k] + st.rc;
#pragma unroll
            for (int q = 0; q < D; ++q) a = fmaf(st.x[q], y[q][k], a);
            t[k] = a;
            e[k] = ex2_approx(a);
        }
        float ts = ((e[0] + e[2]) + (e[4] + e[6])) + ((e[1] + e[3]) + (e[5] + e[7]));
        if (!(ts <= BIG) || !(st.sum + ts >= TINY)) {
            float mx = t[0];
#pragma unroll
            for (int k = 1; k < 8; ++k) mx = fmaxf(mx, t[k]);
            if (mx > -INFINITY) {
                const float sc = (st.sum > 0.f) ? ex2_approx(-mx) : 0.f;
                st.sum *= sc;
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    st.acc[q].x *= sc;
                    st.acc[q].y *= sc;
                }
                st.rc -= mx;
#pragma unroll
                for (int k = 0; k < 8; ++k) e[k] = ex2_approx(t[k] - mx);
                ts = ((e[0] + e[2]) + (e[4] + e[6])) + ((e[1] + e[3]) + (e[5] + e[7]));
            }
        }
        st.sum += ts;
        if constexpr (BARY) {
#pragma unroll
            for (int q = 0; q < D; ++q)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    st.acc[q].x = fmaf(e[2 * u], y[q][2 * u], st.acc[q].x);
                    st.acc[q].y = fmaf(e[2 * u + 1], y[q][2 * u + 1], st.acc[q].y);
                }
        }
    }
    return st;
}

// The rows of one pass are split evenly over the RG row groups (contiguous
// runs, counts differing by at most one); every warp runs the template for its
// own row count, so padding rows cost nothing outside the warps that mix two
// group sizes.  res slot of (group g, row r): g * nrs + r.
struct RsPassMap {
    int lo, q, rem, nrs;  // first row, rows per group (base), groups with one more, stride
    __device__ __forceinline__ int count(int g) const { return q + (g < rem ? 1 : 0); }
    __device__ __forceinline__ int start(int g) const { return lo + g * q + min(g, rem); }
};

template <int D, int NR, bool BARY, class Rows>
__device__ __forceinline__ void rs_rows(const RsCols& cols, int cg_log, const RsPassMap& pm,
                                        const Rows& rows, RsRes* res, RsRes* xw) {
    const int tid = threadIdx.x;
    const int CG = 1 << cg_log;
    const int rg = tid >> cg_log, cg = tid & (CG - 1);
    const int g0 = pm.start(rg), gn = pm.count(rg);
    float x[NR][D], rc[NR], sum[NR];
    float2 acc[NR][D];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        // padding row: every term is exp2(-inf) = 0 and the sum stays 1, in range
        sum[r] = 1.f;
        rc[r] = -INFINITY;
#pragma unroll
        for (int q = 0; q < D; ++q) {
            x[r][q] = 0.f;
            acc[r][q] = make_float2(0.f, 0.f);
        }
        if (r < gn) {
            rows.init(g0 + r, x[r], rc[r]);
            sum[r] = 0.f;
        }
    }
    const float4* wv = reinterpret_cast<const float4*>(rs_smem + cols.w);
    const float4* qv[D];
#pragma unroll
    for (int q = 0; q < D; ++q) qv[q] = reinterpret_cast<const float4*>(rs_smem + cols.q[q]);
    const int steps = cols.nqp >> cg_log;  // quads per thread (even)
    // Streaming pass: no per-tile range tests.  The shift estimate keeps the
    // terms near 2^0, so a row sum that ends in [2^-64, 2^120] is accurate
    // (terms below 2^-126 that flush to zero are < 2^-62 of it); a row that
    // ends outside (nothing accumulated, overflow, NaN) is recomputed by the
    // careful pass below -- in practice only in the first sweep of a flow.
    float2 s2[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) s2[r] = make_float2(sum[r], 0.f);
    for (int kk = 0; kk < steps; kk += 2) {
        const int q0 = cg + (kk << cg_log), q1 = q0 + CG;
        float w[8], y[D][8];
        rs_load8<D>(wv, qv, q0, q1, w, y);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const float2 rc2 = make_float2(rc[r], rc[r]);
            float2 e[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float2 t = __fadd2_rn(make_float2(w[2 * u], w[2 * u + 1]), rc2);
#pragma unroll
                for (int q = 0; q < D; ++q)
                    t = __ffma2_rn(make_float2(x[r][q], x[r][q]),
                                   make_float2(y[q][2 * u], y[q][2 * u + 1]), t);
                // one pair in four on the FMA pipe, three on MUFU.EX2
                if (RS_EMU && u == 3) e[u] = rs_ex2_poly2(t);
                else e[u] = make_float2(ex2_approx(t.x), ex2_approx(t.y));
            }
            s2[r] = __fadd2_rn(s2[r], __fadd2_rn(__fadd2_rn(e[0], e[1]), __fadd2_rn(e[2], e[3])));
            if constexpr (BARY) {
#pragma unroll
                for (int q = 0; q < D; ++q)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        acc[r][q] = __ffma2_rn(e[u], make_float2(y[q][2 * u], y[q][2 * u + 1]),
                                               acc[r][q]);
            }
        }
    }
    bool bad = false;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        sum[r] = s2[r].x + s2[r].y;
        bad |= rs_out_of_range(sum[r]);
    }
    if (bad) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            if (!rs_out_of_range(sum[r])) continue;
            if (r < gn) atomicAdd(&g_rs_careful_rows, 1u);
            RsRowState st;
#pragma unroll
            for (int q = 0; q < D; ++q) st.x[q] = x[r][q];
            st.rc = rc[r];
            st = rs_careful<D, BARY>(wv, qv, cg, cg_log, steps, st);
            rc[r] = st.rc;
            sum[r] = st.sum;
#pragma unroll
            for (int q = 0; q < D; ++q) acc[r][q] = st.acc[q];
        }
    }
    // ---- combine the CG partials of each row (warp shuffles) ---------------
    // one max-butterfly for the row keys, one rescale per lane (exactly 1
    // when the lane kept the row's common shift), then plain sum-butterflies;
    // every butterfly step is commutative, so all lanes end bit-identical
    const int lanes = min(CG, 32);
    float kx[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) kx[r] = -rc[r];
    for (int o = lanes >> 1; o > 0; o >>= 1) {
#pragma unroll
        for (int r = 0; r < NR; ++r) kx[r] = fmaxf(kx[r], __shfl_xor_sync(0xffffffffu, kx[r], o));
    }
    float sv[NR], av[NR][D];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const float k = -rc[r];
        const float f = (k == kx[r]) ? 1.f : ex2_approx(k - kx[r]);
        sv[r] = sum[r] * f;
#pragma unroll
        for (int q = 0; q < D; ++q) av[r][q] = (acc[r][q].x + acc[r][q].y) * f;
    }
    for (int o = lanes >> 1; o > 0; o >>= 1) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            sv[r] += __shfl_xor_sync(0xffffffffu, sv[r], o);
#pragma unroll
            for (int q = 0; q < D; ++q) av[r][q] += __shfl_xor_sync(0xffffffffu, av[r][q], o);
        }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const float k = kx[r], s = sv[r];
        const float* a = av[r];
        if ((tid & (lanes - 1)) == 0 && r < gn) {
            RsRes v;
            v.k = k;
            v.s = s;
#pragma unroll
            for (int q = 0; q < D; ++q) v.a[q] = a[q];
            if (CG <= 32) res[rg * pm.nrs + r] = v;
            else xw[(rg * pm.nrs + r) * (CG >> 5) + (cg >> 5)] = v;
        }
    }
}

// After every warp's rs_rows: merge across the warps of a row group (fixed
// order), then one thread per row runs the epilogue.
template <int D, class Rows, class Epi>
__device__ __forceinline__ void rs_finish(int cg_log, const RsPassMap& pm, const Rows& rows,
                                          Epi&& epi, RsRes* res, RsRes* xw, int tag) {
    const int tid = threadIdx.x;
    const int CG = 1 << cg_log;
    const int RG = RS_BLOCK >> cg_log;
    const int slots = RG * pm.nrs;
    RS_MARK(tag + 1);
    __syncthreads();
    if (CG > 32) {
        const int nw = CG >> 5;
        for (int idx = tid; idx < slots; idx += RS_BLOCK) {
            const int g = idx / pm.nrs, r = idx - g * pm.nrs;
            if (r >= pm.count(g)) continue;
            RsRes v = xw[idx * nw];
            for (int wq = 1; wq < nw; ++wq) {
                const RsRes u = xw[idx * nw + wq];
                const float K = fmaxf(v.k, u.k);
                const float f1 = ex2_approx(v.k - K), f2 = ex2_approx(u.k - K);
                v.s = v.s * f1 + u.s * f2;
#pragma unroll
                for (int q = 0; q < D; ++q) v.a[q] = v.a[q] * f1 + u.a[q] * f2;
                v.k = K;
            }
            res[idx] = v;
        }
        __syncthreads();
    }
    RS_MARK(tag + 2);
    for (int idx = tid; idx < slots; idx += RS_BLOCK) {
        const int g = idx / pm.nrs, r = idx - g * pm.nrs;
        if (r < pm.count(g)) {
            const int li = pm.start(g) + r;
            const RsRes v = res[idx];
            // S is in [2^-64, 2^110]: the MUFU log2 is accurate to ~1e-6 absolute
            const float inv_s = 1.f / v.s;
            const double L2 = rows.rowc2(li) + (double)v.k + (double)__log2f(v.s);
            double bar[D];
#pragma unroll
            for (int q = 0; q < D; ++q) bar[q] = (double)(v.a[q] * inv_s);
            epi(li, L2 * kLn2, bar);
        }
    }
    __syncthreads();
}

// reload: (grid groups) the published folded potentials of the columns,
// copied into shared memory before the first pass.  Passes of at most
// RG * pl.nr rows, balanced.
template <int D, bool BARY, class Rows, class Epi>
__device__ __forceinline__ void rs_sweep(const RsCols& cols, int nrows, RsPlan pl, const Rows& rows,
                                         Epi&& epi, RsRes* res, RsRes* xw,
                                         const float* reload = nullptr, int tag = 20) {
    if (reload) rs_reload(cols, reload);
    __syncthreads();
    RS_MARK(tag);
    const int RG = RS_BLOCK >> pl.cg;
    const int per = RG * pl.nr;
    const int passes = (nrows + per - 1) / per;
    const int warp = threadIdx.x >> 5;
    // first row group of this warp (groups are contiguous runs of CG threads)
    const int wg = pl.cg >= 5 ? (threadIdx.x >> pl.cg) : (warp << (5 - pl.cg));
    for (int p = 0; p < passes; ++p) {
        RsPassMap pm;
        pm.lo = (int)((long long)nrows * p / passes);
        const int cnt = (int)((long long)nrows * (p + 1) / passes) - pm.lo;
        pm.q = cnt / RG;
        pm.rem = cnt - pm.q * RG;
        pm.nrs = pm.q + (pm.rem > 0 ? 1 : 0);
        const int nrw = pm.count(wg);  // warp-uniform: the warp's first group has the most rows
        switch (nrw) {
#define RS_NR(K)                                                                  \
    case K:                                                                       \
        if constexpr (K <= RsMaxNr<D, BARY>::value)                               \
            rs_rows<D, K, BARY>(cols, pl.cg, pm, rows, res, xw);                  \
        break;
            RS_NR(1) RS_NR(2) RS_NR(3) RS_NR(4) RS_NR(5) RS_NR(6) RS_NR(7) RS_NR(8)
#undef RS_NR
            default: break;
        }
        rs_finish<D>(pl.cg, pm, rows, epi, res, xw, tag);
    }
}

// Row sources.  x' = p - c (float), rowc2 = -sd |x'|^2 (double), shift from
// the row's own current potential: log2e (logw - pot / w) (none: 0).
// Own-row cache in shared memory (grid groups; the slices are small): the
// centred coordinates and rowc2 are fixed for a solve, the potential and the
// row shift rc are refreshed by the epilogue that computes the new potential,
// so a pass starts without global loads.
struct RsCache {
    double rowc2, pot;
    float x[3];
    float rc;
};

template <int D>
struct RsRows {
    const double* P;   // points of the sweep's row set
    int base;          // first global row of the slice
    const double* c;   // centre [3]
    double sd;         // log2e / omega
    const double* pot; // nullable (no cache): current potential of the rows
    double logw, inv_w;
    RsCache* cache;    // nullable
    __device__ __forceinline__ double rowc2_global(int li) const {
        const double* p = P + (size_t)(base + li) * D;
        double nrm = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) {
            const double v = p[q] - c[q];
            nrm += v * v;
        }
        return -sd * nrm;
    }
    __device__ __forceinline__ double rowc2(int li) const {
        return cache ? cache[li].rowc2 : rowc2_global(li);
    }
    __device__ __forceinline__ double potential(int li) const {
        return cache ? cache[li].pot : __ldcg(pot + base + li);
    }
    // the row's LSE estimate from a potential; a non-finite potential (an
    // estimate taken from stale memory) means no estimate -- the careful pass
    // then finds the shift, so an estimate never changes a result
    __device__ __forceinline__ double shift2(double pv) const {
        const double e = kLog2e * (logw - pv * inv_w);
        return isfinite(e) ? e : 0.0;
    }
    __device__ __forceinline__ void init(int li, float* x, float& rc) const {
        if (cache) {
            const RsCache& e = cache[li];
#pragma unroll
            for (int q = 0; q < D; ++q) x[q] = e.x[q];
            rc = e.rc;
            return;
        }
        const double* p = P + (size_t)(base + li) * D;
        double nrm = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) {
            const double v = p[q] - c[q];
            x[q] = (float)v;
            nrm += v * v;
        }
        const double est = pot ? shift2(__ldcg(pot + base + li)) : 0.0;
        rc = (float)(-sd * nrm - est);
    }
    // the row's next potential (epilogue): refresh the cached shift
    __device__ __forceinline__ void set_next(int li, double pv) const {
        if (cache) {
            RsCache& e = cache[li];
            e.pot = pv;
            e.rc = (float)(e.rowc2 - shift2(pv));
        }
    }
    // fill the cache for the slice (pot0 nullable: no shift estimate)
    __device__ __forceinline__ void fill(int cnt, const double* pot0) const {
        for (int li = threadIdx.x; li < cnt; li += RS_BLOCK) {
            RsCache e;
            const double* p = P + (size_t)(base + li) * D;
            double nrm = 0.0;
            e.x[0] = e.x[1] = e.x[2] = 0.f;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double v = p[q] - c[q];
                e.x[q] = (float)v;
                nrm += v * v;
            }
            e.rowc2 = -sd * nrm;
            e.pot = pot0 ? pot0[base + li] : 0.0;
            e.rc = (float)(e.rowc2 - (pot0 ? shift2(e.pot) : 0.0));
            cache[li] = e;
        }
    }
};

// Pack a column set: coordinates 2 sd (p - c) and W = sd pot + rowc2; the
// padding up to nqp quads gets W = -inf.
template <int D>
__device__ __forceinline__ void rs_pack(const RsCols& cs, const double* P, int cnt, const double* c,
                                        double sd, const double* pot) {
    const int c4 = cs.nqp * 4;
#pragma unroll 4
    for (int j = threadIdx.x; j < c4; j += RS_BLOCK) {
        if (j < cnt) {
            double nrm = 0.0;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double v = P[(size_t)j * D + q] - c[q];
                rs_smem[cs.q[q] + j] = (float)(2.0 * sd * (double)(float)v);
                nrm += v * v;
            }
            rs_smem[cs.w + j] = (float)(sd * (pot ? pot[j] : 0.0) - sd * nrm);
        } else {
#pragma unroll
            for (int q = 0; q < D; ++q) rs_smem[cs.q[q] + j] = 0.f;
            rs_smem[cs.w + j] = -INFINITY;
        }
    }
}

// Sums of the coordinates and of |p|^2 (acc[0..D), acc[3]) over this
// thread's points, four independent loads in flight per thread.
template <int D>
__device__ __forceinline__ void rs_moments(const double* P, int cnt, double* acc) {
    for (int i0 = threadIdx.x; i0 < cnt; i0 += 4 * RS_BLOCK) {
        double v[4][D];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * RS_BLOCK;
#pragma unroll
            for (int q = 0; q < D; ++q) v[u][q] = (i < cnt) ? P[(size_t)i * D + q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int q = 0; q < D; ++q) {
                acc[q] += v[u][q];
                acc[3] += v[u][q] * v[u][q];
            }
        }
    }
}

// Sum of v[0..n) by one full warp: lane l adds v[l], v[l+32], ... in order,
// then a fixed xor butterfly -- deterministic, and the loads are in flight
// together.  Every lane of the warp must call it; all get the result.
__device__ __forceinline__ double rs_ordered_sum(const double* v, int n) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += __ldcg(v + i);
    return warp_sum(s);
}

// Block-wide moments of a point set (sums of coordinates, sum of |p|^2) in a
// fixed order: out[0..D), out[3]; every thread calls it.
template <int D>
__device__ __forceinline__ void rs_block_moments(const double* P, int cnt, double (*red)[8],
                                                 double* out) {
    double acc[4] = {0, 0, 0, 0};
    rs_moments<D>(P, cnt, acc);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double v = warp_sum(acc[k]);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double v = 0.0;
        for (int w = 0; w < RS_WARPS; ++w) v += red[w][threadIdx.x];
        out[threadIdx.x] = v;
    }
    __syncthreads();
}

__device__ __forceinline__ double rs_nanmax(double a, double b) { return (b > a || b != b) ? b : a; }

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
unsigned next_launch_epoch();  // flow_resident.cu

// Grid groups: CTA 0 resets the barrier and done counters of a launch and
// publishes the launch epoch; the others wait for it before their first
// arrival, so no host-side memset is needed between launches.
__device__ __forceinline__ void rs_start_epoch(const RsArgs& A) {
    if (threadIdx.x == 0) rs_bar_gen = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.bar->count = 0ull;
        *A.done = 0u;
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&A.bar->work), "r"(A.launch_id)
                     : "memory");
    }
}
__device__ __forceinline__ void rs_wait_epoch(const RsArgs& A) {
    if (blockIdx.x != 0 && threadIdx.x == 0) {
        while (ld_acquire_u32(&A.bar->work) != A.launch_id) __nanosleep(32);
    }
}

// The whole flow for one problem (grid group) or for problem blockIdx.x (CTA
// group).  wait_epoch: (grid groups) wait for CTA 0's launch epoch before the
// first barrier (first flow of a launch).
template <int D, bool GRID>
__device__ __forceinline__ void rs_flow_body(const RsArgs& A, bool wait_epoch) {
    __shared__ double s_red[RS_WARPS][8];
    __shared__ double s_sum[8];
    __shared__ RsRes s_res[RS_BLOCK];
    __shared__ RsRes s_xw[RS_WARPS * 8];
    __shared__ int s_last;

    // problem and group
    const int b = GRID ? 0 : (int)blockIdx.x;
    const RsGroup<GRID> grp{GRID ? (int)blockIdx.x : 0, GRID ? (int)gridDim.x : 1, A.bar};
    const int n = A.n, m = A.m;
    const double* X = A.X + (size_t)b * n * D;
    const double* Y = A.Y + (size_t)b * m * D;
    int* plan_state = A.plan_state ? A.plan_state + 8 * b : nullptr;
    if (plan_state && *((volatile const int*)plan_state) != 0) return;
    double* fbuf = A.fbuf + (size_t)b * 2 * n;
    double* pbuf = A.pbuf + (size_t)b * 2 * n;
    double* gbuf = A.gbuf + (size_t)b * m;
    double* dx = A.dx + (size_t)b * n;
    double* dp = A.dp + (size_t)b * n;
    double* bx = A.bx + (size_t)b * n * (D + 1);
    double* bp = A.bp + (size_t)b * n * (D + 1);
    unsigned long long* errslot = A.errslot + 4 * b;
    double* warm_f = A.warm_f ? A.warm_f + (size_t)b * n : nullptr;
    double* warm_p = A.warm_p ? A.warm_p + (size_t)b * n : nullptr;
    int* warm_valid = A.warm_valid ? A.warm_valid + 2 * b : nullptr;
    double* flow = A.flow + (size_t)b * n * D;
    double* fstat = A.fstat + 8 * b;
    double* flow_log = A.flow_log ? A.flow_log + (size_t)b * A.log_stride : nullptr;
    const int tid = threadIdx.x;
    RS_MARK(0);

    // ---- statistics (every CTA, fixed order) -> omega, centres -------------
    // (A.ystat: the target statistics, fixed across the flows of a planner
    // launch, computed once by the caller with this same reduction)
    rs_block_moments<D>(X, n, s_red, s_sum);
    if (A.ystat) {
        if (tid < 4) s_sum[4 + tid] = A.ystat[tid];
        __syncthreads();
    } else {
        rs_block_moments<D>(Y, m, s_red, s_sum + 4);
    }
    double mx[3] = {0, 0, 0}, my[3] = {0, 0, 0}, dot = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
        mx[q] = s_sum[q] / n;
        my[q] = s_sum[4 + q] / m;
        dot += mx[q] * my[q];
    }
    double w = A.omega_fixed;
    if (!(w > 0.0)) {  // resolve_omega "auto" (sinkhorn.py:136-148)
        w = RS_AUTO_OMEGA * (s_sum[3] / n + s_sum[7] / m - 2.0 * dot);
        if (!(w >= RS_OMEGA_FLOOR)) w = (w != w) ? w : RS_OMEGA_FLOOR;
    }
    const double sd = kLog2e / w, inv_w = 1.0 / w;
    const double loga = -log((double)n), logb = -log((double)m);
    double cA[3] = {0, 0, 0}, cB[3] = {0, 0, 0};
#pragma unroll
    for (int q = 0; q < D; ++q) {
        cA[q] = 0.5 * (mx[q] + my[q]);
        cB[q] = mx[q];
    }
    const bool vf = warm_valid && warm_f && warm_valid[0] != 0;
    const bool vp = warm_valid && warm_p && warm_valid[1] != 0;

    // ---- shared-memory column sets -----------------------------------------
    // A: X (centre cA); B: Y (centre cA), later X (centre cB)
    RsCols colA, colB;
    {
        int off = 0;
        for (int q = 0; q < 3; ++q) {
            colA.q[q] = off;
            if (q < D) off += A.ldA;
        }
        colA.w = off;
        off += A.ldA;
        for (int q = 0; q < 3; ++q) {
            colB.q[q] = off;
            if (q < D) off += A.ldB;
        }
        colB.w = off;
    }
    colA.nq = (n + 3) >> 2;
    colA.nqp = A.nqpA;
    colB.nq = (m + 3) >> 2;
    colB.nqp = A.nqpB;
    rs_pack<D>(colA, X, n, cA, sd, vf ? warm_f : nullptr);
    rs_pack<D>(colB, Y, m, cA, sd, nullptr);
    // own row slices
    const int xi0 = (int)((long long)n * grp.rank / grp.size);
    const int xn = (int)((long long)n * (grp.rank + 1) / grp.size) - xi0;
    const int yj0 = (int)((long long)m * grp.rank / grp.size);
    const int yn = (int)((long long)m * (grp.rank + 1) / grp.size) - yj0;
    for (int li = tid; li < xn; li += RS_BLOCK) {
        fbuf[xi0 + li] = vf ? warm_f[xi0 + li] : 0.0;
        pbuf[xi0 + li] = vp ? warm_p[xi0 + li] : 0.0;
    }
    // own-row caches (grid groups): after the column sets in shared memory
    RsCache* cacheY = nullptr;
    RsCache* cacheX = nullptr;
    RsCache* cacheS = nullptr;
    if (A.cache_rows > 0) {
        RsCache* cbase = reinterpret_cast<RsCache*>(rs_smem + A.cache_off);
        cacheY = cbase;
        cacheX = cbase + yn;
        cacheS = cbase + yn + xn;
        // no estimate for sweep A's first pass (g does not exist yet; an
        // estimate from stale memory would make results depend on it)
        RsRows<D>{Y, yj0, cA, sd, nullptr, logb, inv_w, cacheY}.fill(yn, nullptr);
        RsRows<D>{X, xi0, cA, sd, nullptr, loga, inv_w, cacheX}.fill(xn, vf ? warm_f : nullptr);
        RsRows<D>{X, xi0, cB, sd, nullptr, loga, inv_w, cacheS}.fill(xn, vp ? warm_p : nullptr);
    }
    if (GRID && grp.rank == 0) {  // padding of the published arrays
        for (int i = n + tid; i < colA.nq * 4; i += RS_BLOCK) A.WX[i] = -INFINITY;
        for (int j = m + tid; j < colB.nq * 4; j += RS_BLOCK) A.WY[j] = -INFINITY;
        for (int i = n + tid; i < colA.nq * 4; i += RS_BLOCK) A.WY[i] = -INFINITY;
    }
    if (!GRID || grp.rank == 0) {  // padding of the self term's published buffers
        float* WSb = A.WS + (size_t)b * 2 * A.ldWS;
        for (int i = n + tid; i < A.ldWS; i += RS_BLOCK) {
            WSb[i] = -INFINITY;
            WSb[A.ldWS + i] = -INFINITY;
        }
    }
    if (tid == 0 && (!GRID || grp.rank == 0)) {
        errslot[0] = 0ull;
        errslot[1] = 0ull;
        errslot[2] = 0ull;
    }
    if (GRID && wait_epoch) rs_wait_epoch(A);
    __syncthreads();
    RS_MARK(1);
    grp.sync();  // own potentials and error slots visible
    RS_MARK(2);

    // ---- asymmetric solve (X vs Y, sinkhorn.py:170-205) ---------------------
    int cur = 0, it = 0;
    double errA = 0.0;
    bool convA = false;
    while (true) {
        ++it;
        double* fcur = fbuf + (size_t)cur * n;
        double* fnxt = fbuf + (size_t)(cur ^ 1) * n;
        unsigned long long* slot = errslot + (it % 3);
        // sweep A: rows = own Y slice, columns X (potential f)
        {
            const RsRows<D> rows{Y, yj0, cA, sd, it > 1 ? gbuf : nullptr, logb, inv_w, cacheY};
            float* wY = GRID ? A.WY : rs_smem + colB.w;
            rs_sweep<D, false>(colA, yn, A.plA, rows,
                               [&](int li, double L, const double*) {
                                   const int j = yj0 + li;
                                   const double g = w * (logb - L);
                                   gbuf[j] = g;
                                   wY[j] = (float)(sd * g + rows.rowc2(li));
                                   rows.set_next(li, g);
                               },
                               s_res, s_xw, (GRID && it > 1) ? A.WX : nullptr);
        }
        RS_MARK(3);
        grp.sync();
        RS_MARK(4);
        RS_MARK(5);
        // sweep B: rows = own X slice, columns Y (potential g)
        double emax = 0.0;
        {
            const RsRows<D> rows{X, xi0, cA, sd, fcur, loga, inv_w, cacheX};
            float* wX = GRID ? A.WX : rs_smem + colA.w;
            const double csc = 2.0 * sd;
            rs_sweep<D, true>(colB, xn, A.plB, rows,
                              [&](int li, double L, const double* bar) {
                                  const int i = xi0 + li;
                                  const double fi = rows.potential(li);
                                  const double upd = w * (loga - L);
                                  double delta = (fi - upd) * inv_w;
                                  if (delta > RS_EXP_CLIP) delta = RS_EXP_CLIP;
                                  emax = rs_nanmax(emax, fabs(expm1(delta)));
                                  // row sums exp(delta + log a) and the plan row
                                  // mass exp(f / w + L) are formed once, at the end
                                  dx[i] = delta;
                                  double* o = bx + (size_t)i * (D + 1);
                                  o[0] = fi * inv_w + L;
#pragma unroll
                                  for (int q = 0; q < D; ++q) o[1 + q] = bar[q] / csc + cA[q];
                                  fnxt[i] = upd;
                                  wX[i] = (float)(sd * upd + rows.rowc2(li));
                                  rows.set_next(li, upd);
                              },
                              s_res, s_xw, GRID ? A.WY : nullptr, 30);
        }
        RS_MARK(6);
        // CTA max of the error, one atomic per CTA
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) emax = rs_nanmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
        if ((tid & 31) == 0) s_red[tid >> 5][0] = emax;
        __syncthreads();
        if (tid == 0) {
            double bm = 0.0;
            for (int k = 0; k < RS_WARPS; ++k) bm = rs_nanmax(bm, s_red[k][0]);
            if (bm != 0.0) atomic_max_nonneg(slot, bm);
            if (!GRID || grp.rank == 0) errslot[(it + 1) % 3] = 0ull;
        }
        RS_MARK(7);
        grp.sync();
        RS_MARK(8);
        const double err = __longlong_as_double((long long)__ldcg(slot)) / n;
        const bool conv = err <= A.tol;
        if (conv || it >= A.max_iters) {
            errA = err;
            convA = conv;
            break;
        }
        cur ^= 1;
    }
    const int itA = it;
    const double* f_out = fbuf + (size_t)cur * n;  // pre-update f (sinkhorn.py:204)

    // ---- self term (X vs X centred on mean X, sinkhorn.py:208-236) ---------
    __syncthreads();
    colB.nq = colA.nq;
    colB.nqp = A.nqpS;
    rs_pack<D>(colB, X, n, cB, sd, vp ? warm_p : nullptr);
    __syncthreads();
    int pc = 0;
    it = 0;
    double errS = 0.0;
    bool convS = false;
    while (true) {
        ++it;
        double* pcur = pbuf + (size_t)pc * n;
        double* pnxt = pbuf + (size_t)(pc ^ 1) * n;
        unsigned long long* slot = errslot + ((itA + it) % 3);
        // The self update reads and writes the same column set, so the new
        // folded potentials always go to a global buffer (double-buffered: a
        // fast CTA must not overwrite what a slow one is still reloading) and
        // are reloaded by the next iteration -- every update of an iteration
        // reads the previous iterate, as sinkhorn.py:225-231 does.
        float* WSb = A.WS + (size_t)b * 2 * A.ldWS;
        float* pub = WSb + (size_t)(it & 1) * A.ldWS;
        const float* prev = WSb + (size_t)((it & 1) ^ 1) * A.ldWS;
        double emax = 0.0;
        {
            const RsRows<D> rows{X, xi0, cB, sd, pcur, loga, inv_w, cacheS};
            float* wX = pub;
            const double csc = 2.0 * sd;
            rs_sweep<D, true>(colB, xn, A.plS, rows,
                              [&](int li, double L, const double* bar) {
                                  const int i = xi0 + li;
                                  const double fi = rows.potential(li);
                                  const double upd = w * (loga - L);
                                  double delta = (fi - upd) * inv_w;
                                  if (delta > RS_EXP_CLIP) delta = RS_EXP_CLIP;
                                  emax = rs_nanmax(emax, fabs(expm1(delta)));
                                  dp[i] = delta;
                                  double* o = bp + (size_t)i * (D + 1);
                                  o[0] = fi * inv_w + L;
#pragma unroll
                                  for (int q = 0; q < D; ++q) o[1 + q] = bar[q] / csc + cB[q];
                                  const double nxt = 0.5 * (fi + upd);
                                  pnxt[i] = nxt;
                                  wX[i] = (float)(sd * nxt + rows.rowc2(li));
                                  rows.set_next(li, nxt);
                              },
                              s_res, s_xw, it > 1 ? prev : nullptr, 40);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) emax = rs_nanmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
        if ((tid & 31) == 0) s_red[tid >> 5][0] = emax;
        __syncthreads();
        if (tid == 0) {
            double bm = 0.0;
            for (int k = 0; k < RS_WARPS; ++k) bm = rs_nanmax(bm, s_red[k][0]);
            if (bm != 0.0) atomic_max_nonneg(slot, bm);
            if (!GRID || grp.rank == 0) errslot[(itA + it + 1) % 3] = 0ull;
        }
        RS_MARK(12);
        grp.sync();
        RS_MARK(13);
        const double err = __longlong_as_double((long long)__ldcg(slot)) / n;
        const bool conv = err <= A.tol;
        if (conv || it >= A.max_iters) {
            errS = err;
            convS = conv;
            break;
        }
        pc ^= 1;
    }
    const int itS = it;
    const double* p_out = pbuf + (size_t)pc * n;
    RS_MARK(14);

    // ---- envelope gradient for the own rows (sinkhorn.py:383-391) ---------
    const double worst = rs_nanmax(errA, errS);
    const bool flow_error = worst > 100.0 * A.tol;
    double norm_acc = 0.0;
    if (!flow_error) {
        for (int li = tid; li < xn; li += RS_BLOCK) {
            const int i = xi0 + li;
            const double* bxi = bx + (size_t)i * (D + 1);
            const double* bpi = bp + (size_t)i * (D + 1);
            const double rcx = exp(__ldcg(dx + i) + loga), rux = exp(__ldcg(bxi));
            const double rcp = exp(__ldcg(dp + i) + loga), rup = exp(__ldcg(bpi));
            double sq = 0.0;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double xv = X[(size_t)i * D + q];
                const double ty = rux * __ldcg(bxi + 1 + q);
                const double px = rup * __ldcg(bpi + 1 + q);
                const double grad = 2.0 * (rcx * xv - ty) - 2.0 * (rcp * xv - px);
                flow[(size_t)i * D + q] = -grad;
                sq += grad * grad;
            }
            norm_acc += sqrt(sq);
            if (warm_f) {
                warm_f[i] = __ldcg(f_out + i);
                warm_p[i] = __ldcg(p_out + i);
            }
        }
    }
    {
        const double v = warp_sum(norm_acc);
        if ((tid & 31) == 0) s_red[tid >> 5][1] = v;
        __syncthreads();
    }
    double* fin_part = A.fin_part + (GRID ? 0 : b);
    if (tid == 0) {
        double blk = 0.0;
        for (int k = 0; k < RS_WARPS; ++k) blk += s_red[k][1];
        int last = 1;
        if (GRID) {
            fin_part[grp.rank] = blk;
            __threadfence();
            const unsigned prev = atomicAdd(A.done, 1u);
            last = prev == (unsigned)grp.size - 1u;
            if (last) __threadfence();
        } else {
            fin_part[0] = blk;
        }
        s_last = last;
    }
    __syncthreads();
    RS_MARK(15);
    if (!s_last || tid >= 32) return;
    // warp-parallel loads, fixed-order combine (a serial loop of dependent L2
    // loads would cost ~0.4 us per CTA)
    const double total = rs_ordered_sum(fin_part, grp.size);
    if (tid != 0) return;
    if (GRID) *A.done = 0u;  // every other CTA has counted: ready for the next flow
    const double mean_mag = total / n;
    fstat[0] = worst;
    fstat[1] = (convA && convS) ? 1.0 : 0.0;
    fstat[2] = flow_error ? 1.0 : 0.0;
    fstat[3] = flow_error ? NAN : mean_mag;
    fstat[4] = w;
    fstat[5] = (double)itA;
    fstat[6] = (double)itS;
    fstat[7] = 0.0;
    if (!flow_error && warm_valid) {
        warm_valid[0] = 1;
        warm_valid[1] = 1;
    }
    if (plan_state) {
        if (flow_error) {
            plan_state[FCB_STATE_STOP] = 2;
            plan_state[FCB_STATE_STAGE] = 2;
            plan_state[FCB_STATE_ITER] = A.iteration;
            plan_state[FCB_STATE_INDEX] = -1;
        } else {
            double* lg = flow_log + 4 * (size_t)A.iteration;
            lg[0] = mean_mag;
            lg[1] = (double)itA;
            lg[2] = (double)itS;
            lg[3] = worst;
            plan_state[FCB_STATE_FLOWS] = A.iteration + 1;
            if (mean_mag < A.conv_tol) plan_state[FCB_STATE_STOP] = 1;
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int rs_max_nr(int d, bool bary) {
    if (d == 3) return bary ? RsMaxNr<3, true>::value : RsMaxNr<3, false>::value;
    return bary ? RsMaxNr<2, true>::value : RsMaxNr<2, false>::value;
}

static int pad_quads(int nq, int cg) {
    const int step = 2 << cg;
    return (nq + step - 1) / step * step;
}

// Thread layout of a sweep of `rows` rows (per CTA, at most) over `cols`
// columns: the (column threads, rows per thread) pair with the least modelled
// time.  Per 8-column step and row a warp issues ~8 MUFU.EX2 (64 SMSP
// cycles) against ~40 other instructions, plus ~14 per step for the loads, so
// the pair loop is MUFU-bound from one row per thread on; what differs is the
// padding waste (rows rounded up to nr, columns to 2 x threads) and the
// combine cost (butterfly levels, cross-warp merge, fp64 epilogue latency).
static RsPlan rs_pick_plan(int rows, int cols, int d, bool bary, int smem_quads_cap,
                           double bfly = 24.0) {
    const int nq = (cols + 3) / 4;
    const int nrmax = rs_max_nr(d, bary);
    double best = 1e300;
    RsPlan pick{5, 1};
    rows = std::max(rows, 1);
    for (int lg = RS_MIN_CG_LOG; lg <= 9; ++lg) {
        const int RG = RS_BLOCK >> lg;
        const int nqp = pad_quads(nq, lg);
        if (nqp > smem_quads_cap) continue;
        const double steps = (double)(nqp >> lg) / 2.0;
        for (int nr = 1; nr <= nrmax; ++nr) {
            const int per = RG * nr;
            const int passes = (rows + per - 1) / per;
            double cost = 0.0;
            for (int p = 0; p < passes; ++p) {
                const int cnt = (int)((long long)rows * (p + 1) / passes) - (int)((long long)rows * p / passes);
                const int q = cnt / RG, rem = cnt - q * RG;
                // per-SMSP load: warp w runs on SMSP w % 4 with the row count of
                // its first group
                double smsp[4] = {0, 0, 0, 0};
                for (int w = 0; w < RS_WARPS; ++w) {
                    const int g = lg >= 5 ? (w << 5) >> lg : w << (5 - lg);
                    const int k = q + (g < rem ? 1 : 0);
                    if (k > 0) smsp[w & 3] += std::max(64.0 * k, 1.25 * (14.0 + 48.0 * k));
                }
                const double load = *std::max_element(smsp, smsp + 4);
                const int kmax = q + (rem > 0 ? 1 : 0);
                const double comb = kmax * (std::min(lg, 5) * bfly + (lg > 5 ? 60.0 : 0.0)) + 2500.0;
                cost += steps * load + comb;
            }
            if (cost < best - 1e-9) {
                best = cost;
                pick = RsPlan{lg, nr};
            }
        }
    }
    return pick;
}

// Tuning override of a sweep's thread layout: "<cg_log>,<rows per thread>"
// (e.g. FCB_RS_PLAN_B=9,4); ignored unless both are in the kernel's range.
static RsPlan rs_plan_override(const char* var, RsPlan pick, int d, bool bary) {
    const char* v = getenv(var);
    int lg = 0, nr = 0;
    if (v && sscanf(v, "%d,%d", &lg, &nr) == 2 && lg >= RS_MIN_CG_LOG && lg <= 9 && nr >= 1 &&
        nr <= rs_max_nr(d, bary))
        return RsPlan{lg, nr};
    return pick;
}


struct RsWs {
    double *fbuf, *pbuf, *gbuf, *dx, *bx, *dp, *bp, *fin_part;
    float *WX, *WY, *WS;
    int ldWS;
    unsigned long long* errslot;
    unsigned* done;
    GridBarrier* bar;
    size_t total;
};

static RsWs rs_layout(int batch, int n, int m, int d, int group, void* ws, size_t bytes) {
    Arena ar(ws, bytes);
    RsWs L{};
    const size_t B = (size_t)batch;
    L.bar = ar.take<GridBarrier>(1);
    L.done = ar.take<unsigned>(32);
    L.errslot = ar.take<unsigned long long>(4 * B);
    L.fin_part = ar.take<double>(std::max<size_t>(group, B));
    L.fbuf = ar.take<double>(B * 2 * n);
    L.pbuf = ar.take<double>(B * 2 * n);
    L.gbuf = ar.take<double>(B * m);
    L.dx = ar.take<double>(B * n);
    L.dp = ar.take<double>(B * n);
    L.bx = ar.take<double>(B * n * (d + 1));
    L.bp = ar.take<double>(B * n * (d + 1));
    const int nw = 4 * std::max((n + 3) / 4, (m + 3) / 4);
    L.WX = ar.take<float>(nw);
    L.WY = ar.take<float>(nw);
    L.ldWS = 4 * ((n + 3) / 4);
    L.WS = ar.take<float>(B * 2 * (size_t)L.ldWS);
    L.total = ar.off + 256;
    return L;
}

static int rs_smem_limit() {
    static int lim = -1;
    if (lim < 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, current_device()) !=
            cudaSuccess)
            v = 0;
        lim = v;
    }
    return lim;
}

// static shared memory of the kernel (s_red, s_sum, s_res, s_xw) + margin
constexpr size_t RS_STATIC_SMEM = 16 * 1024;

// Full launch configuration of one problem shape.
struct RsShape {
    RsPlan A, B, S;
    int nqpA, nqpB, nqpS, ldA, ldB;
    int cache_off, cache_rows;
    size_t smem;
    bool ok;
};

static RsShape rs_shape(int n, int m, int d, int group, bool cache = true) {
    RsShape s{};
    const int lim = rs_smem_limit();
    if (lim <= 0) return s;
    // generous quads cap for the plan search; checked against the limit below
    const int cap = (int)((lim - RS_STATIC_SMEM) / (4 * (d + 1)) / 4);
    const int xr = (n + group - 1) / group, yr = (m + group - 1) / group;
    // cross sweeps: per-row butterfly levels costed at 80 (measured on B200 with
    // scripts/layout_sweep.sh at config 2: A 16x3 / B 64x2 column threads beat
    // the 24-cost picks 32x5 / 128x4 by 0.8 % / 1.7 % of the step); the self
    // sweep keeps 24 (at 80 it would drop to 4 busy warps).  The 80 cost was
    // fit on grid groups only; one-problem-per-CTA launches (group == 1, the
    // batched planner) keep the 24 cost their layouts were measured with.
    const double bfly = group > 1 ? 80.0 : 24.0;
    s.A = rs_plan_override("FCB_RS_PLAN_A", rs_pick_plan(yr, n, d, false, cap, bfly), d, false);
    s.B = rs_plan_override("FCB_RS_PLAN_B", rs_pick_plan(xr, m, d, true, cap, bfly), d, true);
    s.S = rs_plan_override("FCB_RS_PLAN_S", rs_pick_plan(xr, n, d, true, cap), d, true);
    s.nqpA = pad_quads((n + 3) / 4, s.A.cg);
    s.nqpB = pad_quads((m + 3) / 4, s.B.cg);
    s.nqpS = pad_quads((n + 3) / 4, s.S.cg);
    s.ldA = 4 * s.nqpA;
    s.ldB = 4 * std::max(s.nqpB, s.nqpS);
    s.smem = (size_t)(d + 1) * (s.ldA + s.ldB) * sizeof(float);
    s.cache_off = (int)(align_up(s.smem, 32) / sizeof(float));
    s.cache_rows = cache ? yr + 2 * xr : 0;
    s.smem = align_up(s.smem, 32) + (size_t)s.cache_rows * sizeof(RsCache);
    s.ok = s.smem + RS_STATIC_SMEM <= (size_t)lim;
    return s;
}


static void rs_fill(RsArgs& a, const RsWs& L, const RsShape& sh) {
    a.fbuf = L.fbuf;
    a.pbuf = L.pbuf;
    a.gbuf = L.gbuf;
    a.WX = L.WX;
    a.WY = L.WY;
    a.WS = L.WS;
    a.ldWS = L.ldWS;
    a.dx = L.dx;
    a.bx = L.bx;
    a.dp = L.dp;
    a.bp = L.bp;
    a.errslot = L.errslot;
    a.fin_part = L.fin_part;
    a.done = L.done;
    a.bar = L.bar;
    a.plA = sh.A;
    a.plB = sh.B;
    a.plS = sh.S;
    a.nqpA = sh.nqpA;
    a.nqpB = sh.nqpB;
    a.nqpS = sh.nqpS;
    a.ldA = sh.ldA;
    a.ldB = sh.ldB;
    a.cache_off = sh.cache_off;
    a.cache_rows = sh.cache_rows;
}

}  // namespace fcb
