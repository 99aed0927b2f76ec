// sinkhorn.cu -- streamed log-domain entropic OT on sm_100a.
//
// Replaces sinkhorn.py:136-400 of the reference (resolve_omega, _lse_rows,
// _solve_asymmetric, _solve_symmetric, entropic_ot, sinkhorn_divergence,
// sinkhorn_flow).  The reference materialises C (n x m), C^T and Cxx in
// float64 and runs one numpy pass per operation; here a whole solve is ONE
// cooperative persistent kernel:
//
//   phase 0      pack rows/columns (centred coordinates, folded 1/omega)
//   loop
//     sweep A    rows Y, columns X : partial (max, sum) per column chunk
//     merge A    g = w (log b - LSE), column pack of Y for sweep B
//     sweep B    rows X, columns Y : partial (max, sum, barycentre)
//     merge B    f_new, delta, err = max|expm1(delta)|/n (device atomic max),
//                row sums, plan barycentres, column pack of X for sweep A
//     test       err <= tol or it >= max_iters  (grid-uniform branch)
//
// Cost tiles never exist in memory: each (row, column) pair is evaluated in
// registers from a 16-byte column record broadcast out of shared memory.
//
// fp32 path ("expanded" form, log2 units): with x' = x - c, y' = y - c,
//   a_ij = log2e * (pot_j - |x_i - y_j|^2) / w
//        = W_j + x'_i . Yh_j + rowc_i,
//   W_j = s (pot_j - |y'_j|^2), Yh_j = 2 s y'_j, rowc_i = -s |x'_i|^2,
//   s = log2e / w.  A pair costs d+1 FFMA/FADD, one MUFU.EX2 and one FADD:
//   MUFU-bound (16 ex2/clk/SM).  No running max is tracked: each row is
//   shifted by an estimate of its LSE taken from the current potential (exact
//   at the fixed point), and an 8-column sub-tile whose partial sum leaves
//   [2^-64, 2^64] (or is the first mass of the row) takes a rare slow path
//   that re-shifts by the sub-tile max, so exponents never overflow.
//   Column records are read straight from global memory (L1 broadcast,
//   register double buffer): no shared-memory tiles, no per-tile barriers.
// fp64 path ("direct" form, natural units): a_ij = s pot_j - s |x_i-y_j|^2,
//   used for the reference's tight-tolerance known-answer tests.
#include "fcb_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace fcb {

// Tuning knobs (compile-time; see scripts/tune_ot.sh)
#ifndef FCB_TILE
#define FCB_TILE 512     // columns per shared-memory tile
#endif
#ifndef FCB_MINB
#define FCB_MINB 2       // min resident CTAs per SM (register budget)
#endif
#ifndef FCB_MERGE_SPLIT
#define FCB_MERGE_SPLIT 8  // sweep-B row blocks from which g is merged in its own pass
#endif
#ifndef FCB_EMU_EX2
#define FCB_EMU_EX2 0    // 1: one column pair in four takes 2^t on the FMA pipe (ex2_poly2)
#endif
#ifndef FCB_SAMPLE
#define FCB_SAMPLE 32    // sampled columns per item for the cold-sweep row shift
#endif
#ifndef FCB_OT_SCALAR
#define FCB_OT_SCALAR 0  // 1: fp32 sweeps use the scalar (careful) loop only
#endif

constexpr int OT_BLOCK = 256;
constexpr int OT_SUB = 8;       // columns per register sub-tile
constexpr int OT_SMAX = 96;     // max column chunks per sweep
constexpr int OT_MIN_CHUNK = 64;
constexpr double EXP_CLIP = 500.0;       // sinkhorn.py:67
constexpr double OMEGA_FLOOR = 1e-12;    // sinkhorn.py:66
constexpr double AUTO_OMEGA_FACTOR = 0.05;  // sinkhorn.py:65


struct Sweep {
    int rows, cols, cols8;   // cols8: columns rounded up to OT_SUB
    int nrb;                 // row blocks
    int nchunks, chunk_len;  // column chunks (chunk_len multiple of OT_SUB)
    int items;
};

template <typename Real>
struct OtArgs {
    int mode, n, m, d;
    const double* X;
    const double* Y;
    const double* scal;
    const double* f0;
    int max_iters;
    double tol, loga, logb;
    Vec4<Real>* rowX;
    Vec4<Real>* rowY;
    Vec4<Real>* colX;
    Vec4<Real>* colY;
    double* fbuf;  // 2*n
    double* gbuf;  // m
    double* pm;    // partial shifts  [nchunks][rows of the sweep]
    Real* ps;      // partial sums    [nchunks][rows]
    Real* pa;      // partial moments [nchunks][d][rows]
    double* pm2;   // second partial set (ASYM: sweep B; SYM: odd iterations)
    Real* ps2;
    Real* pa2;
    Sweep A, B;
    GridBarrier* bar;
    unsigned long long* errslot;  // 3 slots
    double* f_out;
    double* g_out;
    double* rs_out;
    double* stat;
    double* bary;
    const int* gate;
    // SWEEP-mode epilogue (fcb_lse_sweep): out = epi_scale omega (epi_shift - L)
    // when epi_scale != 0, else L; bary_L stores L (not 1) in bary[i][0]
    double epi_scale, epi_shift;
    int bary_L;
    // SWEEP-mode row shift estimate (nullable): L_i ~ row_logw - row_est_i / omega
    const double* row_est;
    double row_logw;
};

// ---------------------------------------------------------------------------
// omega / centring statistics (resolve_omega, sinkhorn.py:136-148)
// ---------------------------------------------------------------------------
constexpr int ST_BLOCK = 256;
constexpr int ST_GRID = 148;

// Both point sets in one launch: blocks [0, gx) cover X, [gx, gx + gy) Y.
__global__ void __launch_bounds__(ST_BLOCK) pair_stats_kernel(const double* __restrict__ X, int n,
                                                             const double* __restrict__ Y, int m,
                                                             int d, int gx, double* __restrict__ part) {
    __shared__ double scratch[32];
    const bool isY = (int)blockIdx.x >= gx;
    const double* P = isY ? Y : X;
    const int cnt = isY ? m : n;
    const int nb = isY ? (int)gridDim.x - gx : gx;
    const int b = isY ? (int)blockIdx.x - gx : (int)blockIdx.x;
    double acc[4] = {0, 0, 0, 0};
    const int per = (cnt + nb - 1) / nb;
    const int lo = b * per, hi = min(cnt, lo + per);
    for (int i = lo + threadIdx.x; i < hi; i += ST_BLOCK) {
        double sq = 0.0;
        for (int k = 0; k < d; ++k) {
            const double v = P[(size_t)i * d + k];
            acc[k] += v;
            sq += v * v;
        }
        acc[3] += sq;
    }
    for (int k = 0; k < 4; ++k) {
        const double r = block_sum<ST_BLOCK>(acc[k], scratch);
        if (threadIdx.x == 0) part[blockIdx.x * 4 + k] = r;
    }
}

// omega + centring (resolve_omega, sinkhorn.py:136-148), optionally the
// self-term scal (centre = mean X) and the warm-start selection of
// sinkhorn_flow (sinkhorn.py:364, :371), in one block.  Fixed-order sums.
constexpr int PREP_BLOCK = 1024;
__global__ void __launch_bounds__(PREP_BLOCK)
    flow_prep_kernel(const double* __restrict__ part, int gx, int gy, int n, int m, int d, int mode,
                     double omega_fixed, double unit, double* __restrict__ scal,
                     double* __restrict__ scal_self, const double* __restrict__ warm_f,
                     const double* __restrict__ warm_p, const int* __restrict__ warm_valid,
                     double* __restrict__ f0, double* __restrict__ p0, unsigned* zero_count) {
    __shared__ double scratch[32];
    __shared__ double sums[8];
    for (int k = 0; k < 8; ++k) {
        const int base = (k < 4) ? 0 : gx;
        const int cnt = (k < 4) ? gx : gy;
        double a = 0.0;
        for (int b = threadIdx.x; b < cnt; b += PREP_BLOCK) a += part[(base + b) * 4 + (k & 3)];
        a = block_sum<PREP_BLOCK>(a, scratch);
        if (threadIdx.x == 0) sums[k] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const bool haveY = gy > 0;
        double mx[3] = {0, 0, 0}, my[3] = {0, 0, 0};
        for (int k = 0; k < d; ++k) {
            mx[k] = sums[k] / n;
            my[k] = haveY ? sums[4 + k] / m : mx[k];
        }
        const double mx2 = sums[3] / n;
        const double my2 = haveY ? sums[7] / m : mx2;
        double dot = 0.0;
        for (int k = 0; k < d; ++k) dot += mx[k] * my[k];
        double w = omega_fixed;
        if (!(omega_fixed > 0.0)) {
            w = AUTO_OMEGA_FACTOR * (mx2 + my2 - 2.0 * dot);
            if (!(w >= OMEGA_FLOOR)) w = (w != w) ? w : OMEGA_FLOOR;
        }
        scal[SC_OMEGA] = w;
        scal[SC_S] = unit / w;
        for (int k = 0; k < 3; ++k) {
            double c = 0.0;
            if (k < d) c = (mode == FCB_OT_SYM) ? mx[k] : 0.5 * (mx[k] + my[k]);
            scal[SC_C + k] = c;
            scal[SC_MX + k] = mx[k];
            scal[SC_MY + k] = my[k];
        }
        scal[SC_MX2] = mx2;
        scal[SC_MY2] = my2;
        if (zero_count) *zero_count = 0u;
        if (scal_self) {
            for (int k = 0; k < 16; ++k) scal_self[k] = scal[k];
            for (int k = 0; k < 3; ++k) scal_self[SC_C + k] = (k < d) ? mx[k] : 0.0;
        }
    }
    if (f0) {
        const bool vf = warm_valid && warm_valid[0] != 0;
        const bool vp = warm_valid && warm_valid[1] != 0;
        for (int i = threadIdx.x; i < n; i += PREP_BLOCK) {
            f0[i] = vf ? warm_f[i] : 0.0;
            p0[i] = vp ? warm_p[i] : 0.0;
        }
    }
}

static int stats_blocks(int cnt) { return std::max(1, std::min(ST_GRID, (cnt + 4 * ST_BLOCK - 1) / (4 * ST_BLOCK))); }

// ---------------------------------------------------------------------------
// sweep: one work item = (row block, column chunk)
// ---------------------------------------------------------------------------
template <typename Real>
__device__ __forceinline__ double dexpu(double x) {
    // merge-phase rescale factors: the float path only needs float accuracy
    if constexpr (sizeof(Real) == 4) return (double)ex2_approx((float)x);
    else return exp(x);
}

// Per-row shift estimate for a sweep, from the current potential of the
// row's own point set: at the Sinkhorn fixed point the row LSE equals
// log(a) - pot_i / w exactly (sinkhorn.py:14-15), so shifting by it keeps
// every term near 2^0 and the running max is never tracked.
struct ShiftEst {
    const double* pot;  // nullable: no estimate (shift 0, slow path fixes it)
    double logw;        // log a (rows X) or log b (rows Y)
    double inv_w;       // 1 / omega
    double unit;        // exponent units per natural unit
    __device__ __forceinline__ double at(int i) const {
        if (!pot) return 0.0;
        const double v = unit * (logw - __ldcg(pot + i) * inv_w);
        return isfinite(v) ? v : 0.0;  // a stale/garbage estimate only costs speed
    }
};

template <typename Real>
__device__ __forceinline__ Vec4<Real> load_col(const Vec4<Real>* p) {
    // L1-cacheable broadcast load (every lane of the warp reads the same
    // record).  Columns rewritten by other CTAs are only read after a grid
    // barrier, whose gpu-scope fence makes them visible.
    const Real* q = reinterpret_cast<const Real*>(p);
    return Vec4<Real>{__ldcg(q), __ldcg(q + 1), __ldcg(q + 2), __ldcg(q + 3)};
}

// Column record sources of a sweep.  PlainCols reads packed records;
// MergedCols (sweep B of the asymmetric solve) folds the previous sweep's
// merge into the tile staging: the potential of column j, g_j = w (log b -
// LSE_j), is combined from sweep A's chunk partials of row j right where the
// record is needed -- no merge phase, no grid barrier between the sweeps.
// Every CTA combines the partials in the same order, so all copies of g_j
// are bit-identical; the row-block-0 items also store g.
template <typename Real>
struct PlainCols {
    const Vec4<Real>* cols;
    __device__ __forceinline__ Vec4<Real> operator()(int j) const { return load_col(cols + j); }
    __device__ __forceinline__ PlainCols for_block(int) const { return *this; }
};

template <typename Real>
struct MergedCols {
    const Vec4<Real>* colY;  // packed coordinates (.w unused)
    const Vec4<Real>* rowY;  // .w: row constant of Y
    const double* pm;        // sweep A partials [nch][ldp]
    const Real* ps;
    int nch, ldp, m;
    double w, logb, sd;
    double* gbuf;            // g store (row-block-0 items only)
    double* gout;
    __device__ __forceinline__ Vec4<Real> operator()(int j) const {
        Vec4<Real> c = load_col(colY + j);
        if (j >= m) return c;  // padding record (w = -inf)
        double M = -INFINITY, S = 0.0;
        for (int k = 0; k < nch; ++k) {
            const double mk = __ldcg(pm + (size_t)k * ldp + j);
            const double sk = (double)__ldcg(ps + (size_t)k * ldp + j);
            if (mk > M) {
                const double sc = (S > 0.0) ? dexpu<Real>(M - mk) : 0.0;
                S = S * sc + sk;
                M = mk;
            } else {
                S += sk * dexpu<Real>(mk - M);
            }
        }
        const double L = (M + Units<Real>::logu(S)) / Units<Real>::unit;
        const double g = w * (logb - L);
        if (gout) gout[j] = g;
        c.w = (Real)(sd * g + (double)__ldcg(reinterpret_cast<const Real*>(rowY + j) + 3));
        return c;
    }
    __device__ __forceinline__ MergedCols for_block(int rb) const {
        MergedCols c = *this;
        c.gout = (rb == 0) ? gbuf : nullptr;
        return c;
    }
};

// One work item: RPT rows per thread x columns [c0, c1) (c1 - c0 a multiple
// of OT_SUB).  Emits the partial (shift, sum[, moments]) of every row.
template <typename Real, int D, int RPT, bool EXP, bool BARY, class Cols>
__device__ __forceinline__ void sweep_item(const Vec4<Real>* __restrict__ rows, int nrows, int row0,
                                           const Cols& cols, int c0, int c1,
                                           Vec4<Real>* __restrict__ s_tile,
                                           Real s, const ShiftEst& est, double* __restrict__ pm,
                                           Real* __restrict__ ps, Real* __restrict__ pa, int ldp,
                                           int chunk) {
    using U = Units<Real>;
    const int tid = threadIdx.x;
    const Real BIG = (sizeof(Real) == 4) ? Real(1.8446744e19) : Real(1e150);   // 2^64
    const Real TINY = (sizeof(Real) == 4) ? Real(5.421011e-20) : Real(1e-150); // 2^-64
    Real x[RPT][D], rc[RPT], sum[RPT], acc[RPT][D];
    double rowc_d[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int i = min(row0 + r * OT_BLOCK + tid, nrows - 1);
        const Real* rp = reinterpret_cast<const Real*>(rows + i);
        const Vec4<Real> v{__ldcg(rp), __ldcg(rp + 1), __ldcg(rp + 2), __ldcg(rp + 3)};
#pragma unroll
        for (int k = 0; k < D; ++k) x[r][k] = vget(v, k);
        rowc_d[r] = EXP ? (double)v.w : 0.0;
        rc[r] = (Real)(rowc_d[r] - est.at(i));
        sum[r] = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc[r][k] = 0;
    }
    // columns staged through shared memory (coalesced cooperative loads,
    // LDS.128 broadcast reads)
    for (int t0 = c0; t0 < c1; t0 += FCB_TILE) {
    const int tlen = min(FCB_TILE, c1 - t0);
    __syncthreads();
    for (int k = tid; k < tlen; k += OT_BLOCK) s_tile[k] = cols(t0 + k);
    __syncthreads();
    for (int c = 0; c < tlen; c += OT_SUB) {
        Real cy[OT_SUB][D], cw[OT_SUB];
#pragma unroll
        for (int k = 0; k < OT_SUB; ++k) {
            const Vec4<Real> v = s_tile[c + k];
#pragma unroll
            for (int q = 0; q < D; ++q) cy[k][q] = vget(v, q);
            cw[k] = v.w;
        }
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            Real t[OT_SUB], e[OT_SUB];
#pragma unroll
            for (int k = 0; k < OT_SUB; ++k) {
                if constexpr (EXP) {
                    Real a = cw[k] + rc[r];
#pragma unroll
                    for (int q = 0; q < D; ++q) a = fma(x[r][q], cy[k][q], a);
                    t[k] = a;
                } else {
                    Real d2 = 0;
#pragma unroll
                    for (int q = 0; q < D; ++q) {
                        const Real df = x[r][q] - cy[k][q];
                        d2 = fma(df, df, d2);
                    }
                    t[k] = fma(-s, d2, cw[k] + rc[r]);
                }
                e[k] = U::expu(t[k]);
            }
            Real ts = ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
            if (!(ts <= BIG) || !(sum[r] + ts >= TINY)) {
                // slow path (rare): overflow, NaN, or nothing accumulated yet
                // and the shift estimate is far above this row's terms
                Real mx = t[0];
#pragma unroll
                for (int k = 1; k < OT_SUB; ++k) mx = fmax(mx, t[k]);
                if (mx > Real(-INFINITY)) {
                    const Real sc = (sum[r] > Real(0)) ? U::expu(-mx) : Real(0);
                    sum[r] *= sc;
#pragma unroll
                    for (int q = 0; q < D; ++q) acc[r][q] *= sc;
                    rc[r] -= mx;
#pragma unroll
                    for (int k = 0; k < OT_SUB; ++k) e[k] = U::expu(t[k] - mx);
                    ts = ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
                }
            }
            sum[r] += ts;
            if constexpr (BARY) {
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    Real ta = 0;
#pragma unroll
                    for (int k = 0; k < OT_SUB; ++k) ta = fma(e[k], cy[k][q], ta);
                    acc[r][q] += ta;
                }
            }
        }
    }
    }  // tile loop
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int i = row0 + r * OT_BLOCK + tid;
        if (i < nrows) {
            pm[(size_t)chunk * ldp + i] = rowc_d[r] - (double)rc[r];
            ps[(size_t)chunk * ldp + i] = sum[r];
            if constexpr (BARY) {
#pragma unroll
                for (int q = 0; q < D; ++q) pa[((size_t)chunk * D + q) * ldp + i] = acc[r][q];
            }
        }
    }
}

// fp32 fast path of one work item: columns staged structure-of-arrays
// (w | q0 | q1 | q2 as float4 quads), two columns per packed FADD2/FFMA2,
// one MUFU.EX2 per pair, no per-sub-tile range tests.  The row shift comes
// from the potential estimate, which keeps the terms near 2^0; a row whose
// partial sum ends outside [2^-64, 2^120] (nothing accumulated under a too-high
// shift, overflow, NaN: the first sweep of a cold solve) makes the whole CTA
// redo the item with the careful scalar loop (returns false).  ~5 issue slots
// per pair with barycentres, ~3.5 without: MUFU-bound, where the scalar loop
// (~9.6) was issue-bound.
__device__ __forceinline__ bool f32_out_of_range(float s) {
    constexpr unsigned LO = 0x1F800000u;  // 2^-64
    constexpr unsigned HI = 0x7B800000u;  // 2^120
    return (__float_as_uint(s) - LO) > (HI - LO);
}

template <int D, int RPT, bool BARY, class Cols>
__device__ __forceinline__ bool sweep_item_f32(const Vec4<float>* __restrict__ rows, int nrows,
                                               int row0, const Cols& cols, int c0, int c1,
                                               float* __restrict__ soa, const ShiftEst& est,
                                               double* __restrict__ pm, float* __restrict__ ps,
                                               float* __restrict__ pa, int ldp, int chunk) {
    const int tid = threadIdx.x;
    float x[RPT][D], rc[RPT];
    double rowc_d[RPT];
    float2 s2[RPT], acc[RPT][D];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int i = min(row0 + r * OT_BLOCK + tid, nrows - 1);
        const float* rp = reinterpret_cast<const float*>(rows + i);
        const float4 v = make_float4(__ldcg(rp), __ldcg(rp + 1), __ldcg(rp + 2), __ldcg(rp + 3));
        const float xv[3] = {v.x, v.y, v.z};
#pragma unroll
        for (int q = 0; q < D; ++q) x[r][q] = xv[q];
        rowc_d[r] = (double)v.w;
        rc[r] = (float)(rowc_d[r] - est.at(i));
        s2[r] = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < D; ++q) acc[r][q] = make_float2(0.f, 0.f);
    }
    {
        // shift each row by its max over FCB_SAMPLE columns spread over this
        // item's chunk: the sampled column contributes 2^0, so the partial sum
        // is >= 1 and cannot underflow, and only a chunk whose best column
        // beats the sample's by > ~2^100 overflows (careful loop).  The
        // potential-based estimate is exact only near the fixed point; after a
        // large planner step (config 4 moves the trajectory by hundreds of
        // units per iteration) a warm estimate sends ~15 % of the items to the
        // careful loop, the sample almost none.  Deterministic (fixed columns).
        constexpr int NS = FCB_SAMPLE;
        __syncthreads();
        if (tid < NS) {
            const int span = c1 - c0;
            const Vec4<float> c = cols(c0 + (int)(((long long)span * tid) / NS));
            soa[tid] = c.w;
            soa[NS + tid] = c.x;
            soa[2 * NS + tid] = c.y;
            soa[3 * NS + tid] = c.z;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            float mx = -INFINITY;
            for (int k = 0; k < NS; ++k) {
                float t = soa[k] + (float)rowc_d[r];
                t = fmaf(x[r][0], soa[NS + k], t);
                if (D > 1) t = fmaf(x[r][1], soa[2 * NS + k], t);
                if (D > 2) t = fmaf(x[r][2], soa[3 * NS + k], t);
                mx = fmaxf(mx, t);
            }
            if (mx > -INFINITY && mx < INFINITY) rc[r] = (float)(rowc_d[r] - (double)mx);
        }
    }
    const float4* wv = reinterpret_cast<const float4*>(soa);
    const float4* qv[D];
#pragma unroll
    for (int q = 0; q < D; ++q) qv[q] = reinterpret_cast<const float4*>(soa + (q + 1) * FCB_TILE);
    for (int t0 = c0; t0 < c1; t0 += FCB_TILE) {
        const int tlen = min(FCB_TILE, c1 - t0);
        __syncthreads();
        for (int k = tid; k < tlen; k += OT_BLOCK) {
            const Vec4<float> c = cols(t0 + k);
            soa[k] = c.w;
            soa[FCB_TILE + k] = c.x;
            if (D > 1) soa[2 * FCB_TILE + k] = c.y;
            if (D > 2) soa[3 * FCB_TILE + k] = c.z;
        }
        __syncthreads();
        for (int c = 0; c < tlen; c += OT_SUB) {
            const int q0 = c >> 2, q1 = q0 + 1;
            float w[8], y[D][8];
            {
                const float4 a = wv[q0], b = wv[q1];
                w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
                w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
            }
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const float4 a = qv[q][q0], b = qv[q][q1];
                y[q][0] = a.x; y[q][1] = a.y; y[q][2] = a.z; y[q][3] = a.w;
                y[q][4] = b.x; y[q][5] = b.y; y[q][6] = b.z; y[q][7] = b.w;
            }
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const float2 rc2 = make_float2(rc[r], rc[r]);
                float2 e[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    float2 t = __fadd2_rn(make_float2(w[2 * u], w[2 * u + 1]), rc2);
#pragma unroll
                    for (int q = 0; q < D; ++q)
                        t = __ffma2_rn(make_float2(x[r][q], x[r][q]),
                                       make_float2(y[q][2 * u], y[q][2 * u + 1]), t);
                    if (FCB_EMU_EX2 && u == 3) e[u] = ex2_poly2(t);  // FMA pipe
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
    }
    bool bad = false;
    float sum[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        sum[r] = s2[r].x + s2[r].y;
        if (row0 + r * OT_BLOCK + tid < nrows) bad |= f32_out_of_range(sum[r]);
    }
    if (__syncthreads_or(bad)) return false;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int i = row0 + r * OT_BLOCK + tid;
        if (i < nrows) {
            pm[(size_t)chunk * ldp + i] = rowc_d[r] - (double)rc[r];
            ps[(size_t)chunk * ldp + i] = sum[r];
            if constexpr (BARY) {
#pragma unroll
                for (int q = 0; q < D; ++q)
                    pa[((size_t)chunk * D + q) * ldp + i] = acc[r][q].x + acc[r][q].y;
            }
        }
    }
    return true;
}

// Items that took the careful scalar loop (fp32 fast path refused), for
// fcb_debug_careful_items (diagnostics; one atomic per refused item).
__device__ unsigned g_careful_items;

// All items of a sweep.  Item blockIdx.x is static (no atomic before the
// first item); the rest are handed out dynamically, so CTAs that run faster
// (an SM shared with a slower neighbour, earlier start) take more items.  The
// work counter only grows: a sweep with `items` items consumes exactly
// `items` counter values (every CTA that ran a static item makes one failing
// grab), so the caller advances base by items.  The next item is grabbed
// while the current one runs.
template <typename Real, int D, int RPT, bool EXP, bool BARY, class Cols>
__device__ __forceinline__ void run_sweep(const Sweep& sw, const Vec4<Real>* rows,
                                          const Cols& cols, Real s, const ShiftEst& est,
                                          double* pm, Real* ps, Real* pa, unsigned* work,
                                          unsigned base, Vec4<Real>* s_tile) {
    __shared__ int s_item;
    const int ldp = sw.rows;
    const int grid = gridDim.x;
    int item = blockIdx.x;
    while (item < sw.items) {
        unsigned nxt = 0;
        if (threadIdx.x == 0) nxt = atomicAdd(work, 1u);
        const int rb = item % sw.nrb;
        const int ch = item / sw.nrb;
        const int c0 = ch * sw.chunk_len;
        const int c1 = min(c0 + sw.chunk_len, sw.cols8);
        bool done = false;
        if constexpr (EXP && sizeof(Real) == 4 && !FCB_OT_SCALAR) {
            done = sweep_item_f32<D, RPT, BARY>(rows, sw.rows, rb * OT_BLOCK * RPT,
                                                cols.for_block(rb), c0, c1,
                                                reinterpret_cast<float*>(s_tile), est, pm, ps, pa,
                                                ldp, ch);
        }
        if (!done && EXP && threadIdx.x == 0) atomicAdd(&g_careful_items, 1u);
        if (!done)
            sweep_item<Real, D, RPT, EXP, BARY>(rows, sw.rows, rb * OT_BLOCK * RPT,
                                                cols.for_block(rb), c0, c1, s_tile, s, est, pm, ps,
                                                pa, ldp, ch);
        __syncthreads();
        if (threadIdx.x == 0) s_item = grid + (int)(nxt - base);
        __syncthreads();
        item = s_item;
    }
}

// Merge the column-chunk partials of one row: returns the LSE in natural
// units and, with BARY, the barycentre moments divided by the sum.  G lanes
// of one warp cooperate on one row (G a power of two <= 32); every lane of
// the warp must call this (shuffles use the full mask).
template <typename Real, int D, bool BARY, int G>
__device__ __forceinline__ double merge_row(int i, int nchunks, const double* pm, const Real* ps,
                                            const Real* pa, int ldp, int lane_in_group,
                                            double* bar_out) {
    double M = -INFINITY, S = 0.0, A[D];
#pragma unroll
    for (int q = 0; q < D; ++q) A[q] = 0.0;
    for (int k = lane_in_group; k < nchunks; k += G) {
        const double mk = __ldcg(pm + (size_t)k * ldp + i);
        const double sk = (double)__ldcg(ps + (size_t)k * ldp + i);
        double ak[D];
#pragma unroll
        for (int q = 0; q < D; ++q)
            ak[q] = BARY ? (double)__ldcg(pa + ((size_t)k * D + q) * ldp + i) : 0.0;
        if (mk > M) {
            const double sc = (S > 0.0) ? dexpu<Real>(M - mk) : 0.0;
            S = S * sc + sk;
#pragma unroll
            for (int q = 0; q < D; ++q) A[q] = A[q] * sc + ak[q];
            M = mk;
        } else {
            const double sc = dexpu<Real>(mk - M);
            S += sk * sc;
#pragma unroll
            for (int q = 0; q < D; ++q) A[q] += ak[q] * sc;
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        const double M2 = __shfl_xor_sync(0xffffffffu, M, o);
        const double S2 = __shfl_xor_sync(0xffffffffu, S, o);
        double A2[D];
#pragma unroll
        for (int q = 0; q < D; ++q) A2[q] = __shfl_xor_sync(0xffffffffu, A[q], o);
        const double Mn = fmax(M, M2);
        const double s1 = (S > 0.0) ? dexpu<Real>(M - Mn) : 0.0;
        const double s2 = (S2 > 0.0) ? dexpu<Real>(M2 - Mn) : 0.0;
        // fixed combine order (lower lane's term first): deterministic result
        const bool low = (lane_in_group & o) == 0;
        const double Sa = low ? S * s1 : S2 * s2, Sb = low ? S2 * s2 : S * s1;
        S = Sa + Sb;
#pragma unroll
        for (int q = 0; q < D; ++q) {
            const double Aa = low ? A[q] * s1 : A2[q] * s2, Ab = low ? A2[q] * s2 : A[q] * s1;
            A[q] = Aa + Ab;
        }
        M = Mn;
    }
    if (BARY && bar_out) {
#pragma unroll
        for (int q = 0; q < D; ++q) bar_out[q] = A[q] / S;
    }
    return (M + Units<Real>::logu(S)) / Units<Real>::unit;
}

// A merge phase: rows spread over the whole grid, G lanes per row, warp-
// uniform trip counts.  epi(i, L, bar) runs on the group's lane 0 for valid
// rows only.
template <typename Real, int D, bool BARY, int G, typename Epi>
__device__ __forceinline__ void merge_phase_g(const Sweep& sw, const double* pm, const Real* ps,
                                              const Real* pa, Epi&& epi) {
    constexpr int GPW = 32 / G;  // groups per warp
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int grp = lane / G, lig = lane % G;
    for (int base = warp * GPW; base < sw.rows; base += nwarps * GPW) {
        const int i = base + grp;
        const bool valid = i < sw.rows;
        double bar[D];
        const double L = merge_row<Real, D, BARY, G>(valid ? i : sw.rows - 1, sw.nchunks, pm, ps,
                                                     pa, sw.rows, lig, bar);
        if (valid && lig == 0) epi(i, L, bar);
    }
}

template <typename Real, int D, bool BARY, typename Epi>
__device__ __forceinline__ void merge_phase(const Sweep& sw, const double* pm, const Real* ps,
                                            const Real* pa, Epi&& epi) {
    // G lanes per row: as many as the grid's lanes allow for one pass, but
    // no more than the chunk count needs (grid-uniform choice)
    const long lanes = (long)gridDim.x * blockDim.x;
    int g = 1;
    while (g < 32 && (long)sw.rows * (2 * g) <= lanes && g < sw.nchunks) g <<= 1;
    switch (g) {
        case 1: merge_phase_g<Real, D, BARY, 1>(sw, pm, ps, pa, epi); break;
        case 2: merge_phase_g<Real, D, BARY, 2>(sw, pm, ps, pa, epi); break;
        case 4: merge_phase_g<Real, D, BARY, 4>(sw, pm, ps, pa, epi); break;
        case 8: merge_phase_g<Real, D, BARY, 8>(sw, pm, ps, pa, epi); break;
        case 16: merge_phase_g<Real, D, BARY, 16>(sw, pm, ps, pa, epi); break;
        default: merge_phase_g<Real, D, BARY, 32>(sw, pm, ps, pa, epi); break;
    }
}

// ---------------------------------------------------------------------------
// the persistent solver
// ---------------------------------------------------------------------------
// Scalars of a solve: omega, the exponent scale s = unit / omega and the
// centre (scal[] of resolve_omega, or computed in-kernel by the flow kernel).
struct OtScal {
    double w, sd, c[3];
};

__device__ __forceinline__ OtScal load_scal(const double* scal) {
    return OtScal{scal[SC_OMEGA], scal[SC_S], {scal[SC_C], scal[SC_C + 1], scal[SC_C + 2]}};
}

// Phase 0: centred row records, column records with the folded potential f0
// (nullable), padding, error slots.  Grid-strided; the caller syncs.
template <typename Real, int D>
__device__ __forceinline__ void pack_phase(const OtArgs<Real>& p, const OtScal& sc,
                                           const double* f0) {
    constexpr bool EXP = (sizeof(Real) == 4);
    const double sd = sc.sd;
    const double* c = sc.c;
    const int gthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const bool asym = (p.mode == FCB_OT_ASYM);
    const bool sweep_only = (p.mode == FCB_OT_SWEEP);
    const double csc = EXP ? 2.0 * sd : 1.0;  // column coordinate scale
    for (int i = gtid; i < p.n; i += gthreads) {
        Real xs[3] = {0, 0, 0};
        double nrm = 0.0;
        for (int k = 0; k < D; ++k) {
            const double v = p.X[(size_t)i * D + k] - c[k];
            xs[k] = (Real)v;
            nrm += v * v;
        }
        const double rowc = EXP ? -sd * nrm : 0.0;
        p.rowX[i] = Vec4<Real>{xs[0], xs[1], xs[2], (Real)rowc};
        if (!sweep_only) {
            const double f = f0 ? f0[i] : 0.0;
            p.fbuf[i] = f;
            p.colX[i] = Vec4<Real>{(Real)(csc * (double)xs[0]), (Real)(csc * (double)xs[1]),
                                   (Real)(csc * (double)xs[2]), (Real)(sd * f + rowc)};
        }
    }
    if (!sweep_only) {
        const int pad_end = (p.n + OT_SUB - 1) / OT_SUB * OT_SUB;
        for (int i = p.n + gtid; i < pad_end; i += gthreads)
            p.colX[i] = Vec4<Real>{0, 0, 0, (Real)-INFINITY};
    }
    if (asym || sweep_only) {
        for (int j = gtid; j < p.m; j += gthreads) {
            Real ys[3] = {0, 0, 0};
            double nrm = 0.0;
            for (int k = 0; k < D; ++k) {
                const double v = p.Y[(size_t)j * D + k] - c[k];
                ys[k] = (Real)v;
                nrm += v * v;
            }
            const double rowc = EXP ? -sd * nrm : 0.0;
            if (asym) p.rowY[j] = Vec4<Real>{ys[0], ys[1], ys[2], (Real)rowc};
            const double pot = sweep_only ? f0[j] : 0.0;
            p.colY[j] = Vec4<Real>{(Real)(csc * (double)ys[0]), (Real)(csc * (double)ys[1]),
                                   (Real)(csc * (double)ys[2]), (Real)(sd * pot + rowc)};
        }
        const int pad_end = (p.m + OT_SUB - 1) / OT_SUB * OT_SUB;
        for (int j = p.m + gtid; j < pad_end; j += gthreads)
            p.colY[j] = Vec4<Real>{0, 0, 0, (Real)-INFINITY};
    }
    if (gtid == 0) {
        p.errslot[0] = 0ull;
        p.errslot[1] = 0ull;
        p.errslot[2] = 0ull;
    }
}

// The SWEEP mode: one LSE pass of rows X over columns Y (potential f0).
template <typename Real, int D, int RPT, bool BARY>
__device__ __forceinline__ void sweep_only_pass(const OtArgs<Real>& p, const OtScal& sc,
                                                Vec4<Real>* s_tile) {
    constexpr bool EXP = (sizeof(Real) == 4);
    const Real s = (Real)sc.sd;
    const double* c = sc.c;
    const double csc = EXP ? 2.0 * sc.sd : 1.0;
    const double unit = Units<Real>::unit;
    const ShiftEst est{p.row_est, p.row_logw, 1.0 / sc.w, unit};
    run_sweep<Real, D, RPT, EXP, BARY>(p.B, p.rowX, PlainCols<Real>{p.colY}, s, est, p.pm, p.ps,
                                       p.pa, &p.bar->work, 0u, s_tile);
    grid_sync(p.bar);
    double* out = p.f_out;
    double* bo = p.bary;
    merge_phase<Real, D, BARY>(p.B, p.pm, p.ps, p.pa, [&](int i, double L, const double* bar) {
        if (out) out[i] = (p.epi_scale != 0.0) ? p.epi_scale * sc.w * (p.epi_shift - L) : L;
        if (BARY && bo) {  // weighted mean of the columns (M-shard combine)
            double* o = bo + (size_t)i * (D + 1);
            o[0] = p.bary_L ? L : 1.0;
            for (int q = 0; q < D; ++q) o[1 + q] = bar[q] / csc + c[q];
        }
    });
}

// The Sinkhorn iterations of an ASYM or SYM solve (after pack_phase and a
// grid barrier) up to convergence or max_iters, then the outputs.  wbase:
// work-counter base, carried across solves that share the barrier.
template <typename Real, int D, int RPT, bool BARY>
__device__ __forceinline__ void solve_loop(const OtArgs<Real>& p, const OtScal& sc, unsigned& wbase,
                                           double* red, Vec4<Real>* s_tile) {
    constexpr bool EXP = (sizeof(Real) == 4);
    const double w = sc.w;
    const double sd = sc.sd;
    const Real s = (Real)sd;
    const double* c = sc.c;
    const int gthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const bool asym = (p.mode == FCB_OT_ASYM);
    const double csc = EXP ? 2.0 * sd : 1.0;
    const double unit = Units<Real>::unit;
    const double inv_n = 1.0 / p.n;
    int cur = 0;
    int it = 0;
    while (true) {
        ++it;
        const double* fcur = p.fbuf + (size_t)cur * p.n;
        double* fnxt = p.fbuf + (size_t)(cur ^ 1) * p.n;
        unsigned long long* slot = p.errslot + (it % 3);
        // sweep partials: ASYM sweep A -> set 1, sweep B -> set 2 (sweep B
        // reads set 1 while it runs); SYM -> set 1
        double* pmB = asym ? p.pm2 : p.pm;
        Real* psB = asym ? p.ps2 : p.ps;
        Real* paB = asym ? p.pa2 : p.pa;
        const ShiftEst estB{fcur, p.loga, 1.0 / w, unit};
        if (asym) {
            // ---- sweep A: rows Y, columns X (potential f) --------------
            // shift estimate of the careful loop: g of the previous iteration
            // (none at it == 1); the fp32 fast path samples its own shift
            const ShiftEst estA{it > 1 ? p.gbuf : nullptr, p.logb, 1.0 / w, unit};
            run_sweep<Real, D, RPT, EXP, false>(p.A, p.rowY, PlainCols<Real>{p.colX}, s, estA, p.pm,
                                                p.ps, p.pa, &p.bar->work, wbase, s_tile);
            wbase += (unsigned)p.A.items;
            grid_sync(p.bar);
            // ---- sweep B: rows X, columns Y with g = w (log b - LSE_A) ----
            if (p.B.nrb >= FCB_MERGE_SPLIT) {
                // many row blocks: merge g once per column (one pass, one grid
                // barrier) instead of once per row block in the tile staging
                merge_phase<Real, D, false>(p.A, p.pm, p.ps, p.pa,
                                            [&](int j, double L, const double*) {
                                                const double g = w * (p.logb - L);
                                                p.gbuf[j] = g;
                                                p.colY[j].w = (Real)(sd * g + (double)p.rowY[j].w);
                                            });
                grid_sync(p.bar);
                run_sweep<Real, D, RPT, EXP, BARY>(p.B, p.rowX, PlainCols<Real>{p.colY}, s, estB,
                                                   pmB, psB, paB, &p.bar->work, wbase, s_tile);
            } else {
                // few row blocks: merged from sweep A's partials while staging
                // the tiles (no merge pass, no extra barrier)
                const MergedCols<Real> colsB{p.colY, p.rowY, p.pm, p.ps, p.A.nchunks, p.A.rows,
                                             p.m, w, p.logb, sd, p.gbuf, nullptr};
                run_sweep<Real, D, RPT, EXP, BARY>(p.B, p.rowX, colsB, s, estB, pmB, psB, paB,
                                                   &p.bar->work, wbase, s_tile);
            }
        } else {
            // ---- SYM: rows X, columns X --------------------------------------
            run_sweep<Real, D, RPT, EXP, BARY>(p.B, p.rowX, PlainCols<Real>{p.colX}, s, estB, pmB,
                                               psB, paB, &p.bar->work, wbase, s_tile);
        }
        wbase += (unsigned)p.B.items;
        grid_sync(p.bar);
        // ---- merge B ------------------------------------------------------
        double emax = 0.0;
        merge_phase<Real, D, BARY>(p.B, pmB, psB, paB, [&](int i, double L, const double* bar) {
            const double fi = __ldcg(fcur + i);
            const double upd = w * (p.loga - L);  // f_new (ASYM) / target (SYM)
            double delta = (fi - upd) / w;
            if (delta > EXP_CLIP) delta = EXP_CLIP;  // np.clip(., None, 500); NaN passes
            const double e = fabs(expm1(delta));
            emax = (e > emax || e != e) ? e : emax;
            p.rs_out[i] = exp(delta + p.loga);
            if (BARY && p.bary) {
                double* o = p.bary + (size_t)i * (D + 1);
                o[0] = exp(fi / w + L);
                for (int q = 0; q < D; ++q) o[1 + q] = bar[q] / csc + c[q];
            }
            const double nxt = asym ? upd : 0.5 * (fi + upd);
            fnxt[i] = nxt;
            p.colX[i].w = (Real)(sd * nxt + (double)p.rowX[i].w);
        });
        for (int o = 16; o > 0; o >>= 1) {
            const double v = __shfl_xor_sync(0xffffffffu, emax, o);
            emax = (v > emax || v != v) ? v : emax;
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = emax;
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = 0.0;
            for (int k = 0; k < OT_BLOCK / 32; ++k) b = (red[k] > b || red[k] != red[k]) ? red[k] : b;
            // max with the slot's initial 0 is a no-op: blocks without rows skip
            // the (contended) atomic
            if (b != 0.0) atomic_max_nonneg(slot, b);
            if (blockIdx.x == 0) p.errslot[(it + 1) % 3] = 0ull;
        }
        grid_sync(p.bar);
        const double err = __longlong_as_double((long long)__ldcg(slot)) * inv_n;
        const bool conv = err <= p.tol;
        if (conv || it >= p.max_iters) {
            for (int i = gtid; i < p.n; i += gthreads) p.f_out[i] = __ldcg(fcur + i);
            if (asym && p.g_out)
                for (int j = gtid; j < p.m; j += gthreads) p.g_out[j] = __ldcg(p.gbuf + j);
            if (gtid == 0) {
                p.stat[0] = err;
                p.stat[1] = (double)it;
                p.stat[2] = conv ? 1.0 : 0.0;
                p.stat[3] = 0.0;
            }
            return;
        }
        cur ^= 1;
    }
}

template <typename Real, int D, int RPT, bool BARY>
__global__ void __launch_bounds__(OT_BLOCK, FCB_MINB) ot_solve_kernel(OtArgs<Real> p) {
    __shared__ double red[32];
    __shared__ Vec4<Real> s_tile[FCB_TILE];  // column records of the current tile
    if (p.gate && *((volatile const int*)p.gate) != 0) return;
    const OtScal sc = load_scal(p.scal);
    pack_phase<Real, D>(p, sc, p.f0);
    grid_sync(p.bar);
    if (p.mode == FCB_OT_SWEEP) {
        sweep_only_pass<Real, D, RPT, BARY>(p, sc, s_tile);
        return;
    }
    unsigned wbase = 0;
    solve_loop<Real, D, RPT, BARY>(p, sc, wbase, red, s_tile);
}

// ---------------------------------------------------------------------------
// sinkhorn_flow in one launch (sinkhorn.py:355-397): statistics and omega,
// the packs of both problems, the asymmetric solve (X vs Y), the self term
// (X vs X), the envelope gradient, warm state and planner hooks.  The grid
// barrier and its work counter are shared by both solves.
// ---------------------------------------------------------------------------
template <typename Real>
struct FlowArgs {
    OtArgs<Real> a;  // X vs Y, centred on (mean X + mean Y) / 2
    OtArgs<Real> b;  // X vs X, centred on mean X
    double omega_fixed;
    double* part;      // grid x 8 partial sums (X: sum, |x|^2; Y: same)
    double* scal;      // [16] outputs (resolve_omega layout)
    double* scal_self;
    double* warm_f;    // warm state: read at the start, stored at the end
    double* warm_p;
    int* warm_valid;
    double* flow;
    double* fstat;
    int* plan_state;
    int iteration;
    double* flow_log;
    double conv_tol;
    double* fin_part;  // grid
};

template <typename Real, int D, int RPT>
__global__ void __launch_bounds__(OT_BLOCK, FCB_MINB) flow_kernel(FlowArgs<Real> fa) {
    __shared__ double red[32];
    __shared__ double s_sum[8];
    __shared__ Vec4<Real> s_tile[FCB_TILE];
    const OtArgs<Real>& A = fa.a;
    const OtArgs<Real>& B = fa.b;
    if (fa.plan_state && *((volatile const int*)fa.plan_state) != 0) return;
    const int gthreads = gridDim.x * blockDim.x;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = A.n, m = A.m;

    // ---- statistics of X and Y -> omega and both centrings ----------------
    {
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = gtid; i < n; i += gthreads) {
            double sq = 0.0;
            for (int k = 0; k < D; ++k) {
                const double v = A.X[(size_t)i * D + k];
                acc[k] += v;
                sq += v * v;
            }
            acc[3] += sq;
        }
        for (int j = gtid; j < m; j += gthreads) {
            double sq = 0.0;
            for (int k = 0; k < D; ++k) {
                const double v = A.Y[(size_t)j * D + k];
                acc[4 + k] += v;
                sq += v * v;
            }
            acc[7] += sq;
        }
        for (int k = 0; k < 8; ++k) {
            const double r = block_sum<OT_BLOCK>(acc[k], red);
            if (threadIdx.x == 0) fa.part[blockIdx.x * 8 + k] = r;
        }
    }
    grid_sync(A.bar);
    if (threadIdx.x < 32) {  // every CTA combines the partials in one fixed order
        const int lane = threadIdx.x;
        for (int k = 0; k < 8; ++k) {
            double v = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(fa.part + b * 8 + k);
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) s_sum[k] = v;
        }
    }
    __syncthreads();
    double mx[3] = {0, 0, 0}, my[3] = {0, 0, 0}, dot = 0.0;
    for (int k = 0; k < D; ++k) {
        mx[k] = s_sum[k] / n;
        my[k] = s_sum[4 + k] / m;
        dot += mx[k] * my[k];
    }
    const double mx2 = s_sum[3] / n, my2 = s_sum[7] / m;
    double w = fa.omega_fixed;
    if (!(w > 0.0)) {  // resolve_omega "auto", sinkhorn.py:136-148
        w = AUTO_OMEGA_FACTOR * (mx2 + my2 - 2.0 * dot);
        if (!(w >= OMEGA_FLOOR)) w = (w != w) ? w : OMEGA_FLOOR;
    }
    const double unit = Units<Real>::unit;
    OtScal scA{w, unit / w, {0, 0, 0}}, scB{w, unit / w, {0, 0, 0}};
    for (int k = 0; k < D; ++k) {
        scA.c[k] = 0.5 * (mx[k] + my[k]);
        scB.c[k] = mx[k];
    }
    if (gtid == 0) {
        for (double* sc : {fa.scal, fa.scal_self}) {
            const bool self = sc == fa.scal_self;
            sc[SC_OMEGA] = w;
            sc[SC_S] = unit / w;
            for (int k = 0; k < 3; ++k) {
                sc[SC_C + k] = self ? scB.c[k] : scA.c[k];
                sc[SC_MX + k] = mx[k];
                sc[SC_MY + k] = my[k];
            }
            sc[SC_MX2] = mx2;
            sc[SC_MY2] = my2;
        }
    }
    // warm start: the previous flow's potentials when they were stored
    const bool vf = fa.warm_valid && fa.warm_valid[0] != 0;
    const bool vp = fa.warm_valid && fa.warm_valid[1] != 0;
    pack_phase<Real, D>(A, scA, vf ? fa.warm_f : nullptr);
    pack_phase<Real, D>(B, scB, vp ? fa.warm_p : nullptr);
    grid_sync(A.bar);

    unsigned wbase = 0;
    solve_loop<Real, D, RPT, true>(A, scA, wbase, red, s_tile);
    solve_loop<Real, D, RPT, true>(B, scB, wbase, red, s_tile);
    grid_sync(A.bar);

    // ---- finalize: FlowError test, envelope gradient, warm state ----------
    const double ex = __ldcg(A.stat), ep = __ldcg(B.stat);
    const double worst = (ex > ep || ex != ex) ? ex : ep;
    const bool flow_error = worst > 100.0 * A.tol;
    double norm_acc = 0.0;
    if (!flow_error) {
        for (int i = gtid; i < n; i += gthreads) {
            const double* bx = A.bary + (size_t)i * (D + 1);
            const double* bp = B.bary + (size_t)i * (D + 1);
            const double rcx = __ldcg(A.rs_out + i), rux = __ldcg(bx);
            const double rcp = __ldcg(B.rs_out + i), rup = __ldcg(bp);
            double sq = 0.0;
            for (int k = 0; k < D; ++k) {
                const double x = A.X[(size_t)i * D + k];
                const double ty = rux * __ldcg(bx + 1 + k);
                const double px = rup * __ldcg(bp + 1 + k);
                const double grad = 2.0 * (rcx * x - ty) - 2.0 * (rcp * x - px);
                fa.flow[(size_t)i * D + k] = -grad;
                sq += grad * grad;
            }
            norm_acc += sqrt(sq);
            if (fa.warm_f) {
                fa.warm_f[i] = __ldcg(A.f_out + i);
                fa.warm_p[i] = __ldcg(B.f_out + i);
            }
        }
    }
    const double blk = block_sum<OT_BLOCK>(norm_acc, red);
    if (threadIdx.x == 0) fa.fin_part[blockIdx.x] = blk;
    grid_sync(A.bar);
    if (blockIdx.x != 0) return;
    double tsum = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += OT_BLOCK) tsum += __ldcg(fa.fin_part + b);
    const double total = block_sum<OT_BLOCK>(tsum, red);
    if (threadIdx.x == 0) {
        const double mean_mag = total / n;
        double* fs = fa.fstat;
        fs[0] = worst;
        fs[1] = (__ldcg(A.stat + 2) != 0.0 && __ldcg(B.stat + 2) != 0.0) ? 1.0 : 0.0;
        fs[2] = flow_error ? 1.0 : 0.0;
        fs[3] = flow_error ? NAN : mean_mag;
        fs[4] = w;
        fs[5] = __ldcg(A.stat + 1);
        fs[6] = __ldcg(B.stat + 1);
        fs[7] = 0.0;
        if (!flow_error && fa.warm_valid) {
            fa.warm_valid[0] = 1;
            fa.warm_valid[1] = 1;
        }
        if (int* ps = fa.plan_state) {
            if (flow_error) {
                ps[FCB_STATE_STOP] = 2;
                ps[FCB_STATE_STAGE] = 2;
                ps[FCB_STATE_ITER] = fa.iteration;
                ps[FCB_STATE_INDEX] = -1;
            } else {
                double* lg = fa.flow_log + 4 * (size_t)fa.iteration;
                lg[0] = mean_mag;
                lg[1] = fs[5];
                lg[2] = fs[6];
                lg[3] = worst;
                ps[FCB_STATE_FLOWS] = fa.iteration + 1;
                if (mean_mag < fa.conv_tol) ps[FCB_STATE_STOP] = 1;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static Sweep plan_sweep(int rows, int cols, int rpt, int grid) {
    Sweep s{};
    s.rows = rows;
    s.cols = cols;
    s.cols8 = (cols + OT_SUB - 1) / OT_SUB * OT_SUB;
    const int br = OT_BLOCK * rpt;
    s.nrb = (rows + br - 1) / br;
    const int max_chunks = std::max(1, std::min(OT_SMAX, s.cols8 / OT_MIN_CHUNK));
    const double pairs = (double)rows * (double)cols;
    if (pairs > 4e5 * grid) {
        // large sweeps: several items per CTA (~200k pairs each, at most 8 per
        // CTA), balanced at run time by the dynamic item counter
        const double target = std::min(8.0 * grid, pairs / 2e5);
        const int k = std::max(1, std::min(max_chunks, (int)std::ceil(target / s.nrb)));
        int cl = (s.cols8 + k - 1) / k;
        cl = (cl + OT_SUB - 1) / OT_SUB * OT_SUB;
        s.chunk_len = cl;
        s.nchunks = (s.cols8 + cl - 1) / cl;
        s.items = s.nrb * s.nchunks;
        return s;
    }
    // small sweeps: the chunk count that best fills whole waves of the grid
    int best = 1;
    double best_eff = -1.0;
    for (int k = 1; k <= max_chunks; ++k) {
        const long items = (long)s.nrb * k;
        const long waves = (items + grid - 1) / grid;
        const double eff = (double)items / (double)(waves * grid);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = k;
        }
        if (eff > 0.97) break;
    }
    int cl = (s.cols8 + best - 1) / best;
    cl = (cl + OT_SUB - 1) / OT_SUB * OT_SUB;
    s.chunk_len = cl;
    s.nchunks = (s.cols8 + cl - 1) / cl;
    s.items = s.nrb * s.nchunks;
    return s;
}

template <typename Real>
struct OtLayout {
    size_t bytes = 0;
    OtArgs<Real> a{};
};

template <typename Real, int D, int RPT, bool BARY>
static int ot_grid_size(int* grid) {
    static int cached = -1;
    if (cached < 0) {
        int per_sm = 0;
        FCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, ot_solve_kernel<Real, D, RPT, BARY>, OT_BLOCK, 0));
        if (per_sm < 1) return fail(FCB_ECUDA, "ot_solve_kernel cannot be resident");
        // more resident CTAs hide MUFU/FMA latency but add grid-barrier
        // arrivals; FCB_OT_CTAS_PER_SM overrides the default of 2
        int cap = 2;
        if (const char* env = getenv("FCB_OT_CTAS_PER_SM")) cap = std::max(1, atoi(env));
        per_sm = std::min(per_sm, cap);
        cached = per_sm * sm_count();
    }
    *grid = cached;
    return FCB_OK;
}

template <typename Real>
static void ot_layout(OtLayout<Real>& L, int mode, int n, int m, int d, int rpt, int grid,
                      void* ws, size_t ws_bytes) {
    Arena ar(ws, ws_bytes);
    OtArgs<Real>& a = L.a;
    a.mode = mode;
    a.n = n;
    a.m = m;
    a.d = d;
    const bool asym = mode == FCB_OT_ASYM;
    const bool sweep = mode == FCB_OT_SWEEP;
    a.A = Sweep{};
    if (asym) {
        a.A = plan_sweep(m, n, rpt, grid);
        a.B = plan_sweep(n, m, rpt, grid);
    } else if (sweep) {
        a.B = plan_sweep(n, m, rpt, grid);
    } else {
        a.B = plan_sweep(n, n, rpt, grid);
    }
    const size_t n8 = (size_t)(n + OT_SUB - 1) / OT_SUB * OT_SUB;
    const size_t m8 = (size_t)(m + OT_SUB - 1) / OT_SUB * OT_SUB;
    a.rowX = ar.take<Vec4<Real>>(n);
    a.rowY = ar.take<Vec4<Real>>(asym ? m : 0);
    a.colX = ar.take<Vec4<Real>>(sweep ? 0 : n8);
    a.colY = ar.take<Vec4<Real>>((asym || sweep) ? m8 : 0);
    a.fbuf = ar.take<double>(sweep ? 0 : 2 * (size_t)n);
    a.gbuf = ar.take<double>(asym ? m : 0);
    const size_t pcount = std::max((size_t)a.A.nchunks * a.A.rows, (size_t)a.B.nchunks * a.B.rows);
    a.pm = ar.take<double>(pcount);
    a.ps = ar.take<Real>(pcount);
    a.pa = ar.take<Real>(pcount * d);
    a.pm2 = ar.take<double>(sweep ? 0 : pcount);
    a.ps2 = ar.take<Real>(sweep ? 0 : pcount);
    a.pa2 = ar.take<Real>(sweep ? 0 : pcount * d);
    a.bar = ar.take<GridBarrier>(1);
    a.errslot = ar.take<unsigned long long>(4);
    L.bytes = ar.off + 256;
}

struct OtEpi {
    double scale = 0.0, shift = 0.0;
    int bary_L = 0;
    const double* row_est = nullptr;
    double row_logw = 0.0;
};

template <typename Real, int D, int RPT, bool BARY>
static int ot_launch(int mode, const double* X, int n, const double* Y, int m, const double* scal,
                     int max_iters, double tol, const double* f0, double* f, double* g,
                     double* rs, double* stat, double* bary, const int* gate, void* ws,
                     size_t ws_bytes, cudaStream_t st, OtEpi epi = OtEpi{}) {
    int grid = 0;
    int rc = ot_grid_size<Real, D, RPT, BARY>(&grid);
    if (rc) return rc;
    OtLayout<Real> L;
    ot_layout<Real>(L, mode, n, m, D, RPT, grid, ws, ws_bytes);
    if (L.bytes > ws_bytes) return fail(FCB_EWORKSPACE, "ot workspace too small");
    OtArgs<Real>& a = L.a;
    a.X = X;
    a.Y = Y;
    a.scal = scal;
    a.f0 = f0;
    a.max_iters = max_iters;
    a.tol = tol;
    a.loga = -log((double)n);
    a.logb = (m > 0) ? -log((double)m) : 0.0;
    a.f_out = f;
    a.g_out = g;
    a.rs_out = rs;
    a.stat = stat;
    a.bary = bary;
    a.gate = gate;
    a.epi_scale = epi.scale;
    a.epi_shift = epi.shift;
    a.bary_L = epi.bary_L;
    a.row_est = epi.row_est;
    a.row_logw = epi.row_logw;
    FCB_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(GridBarrier), st));
    void* args[] = {&a};
    FCB_CUDA(cudaLaunchCooperativeKernel((const void*)ot_solve_kernel<Real, D, RPT, BARY>,
                                         dim3(grid), dim3(OT_BLOCK), args, 0, st));
    FCB_LAUNCHED("ot_solve_kernel");
    return FCB_OK;
}

template <typename Real, int RPT>
static int ot_dispatch(int mode, int d, const double* X, int n, const double* Y, int m,
                       const double* scal, int max_iters, double tol, const double* f0, double* f,
                       double* g, double* rs, double* stat, double* bary, const int* gate,
                       void* ws, size_t ws_bytes, cudaStream_t st) {
#define FCB_OT_CASE(DD)                                                                          \
    if (d == DD) {                                                                               \
        if (bary)                                                                                \
            return ot_launch<Real, DD, RPT, true>(mode, X, n, Y, m, scal, max_iters, tol, f0, f, \
                                                  g, rs, stat, bary, gate, ws, ws_bytes, st);    \
        return ot_launch<Real, DD, RPT, false>(mode, X, n, Y, m, scal, max_iters, tol, f0, f, g, \
                                               rs, stat, bary, gate, ws, ws_bytes, st);          \
    }
    FCB_OT_CASE(1)
    FCB_OT_CASE(2)
    FCB_OT_CASE(3)
#undef FCB_OT_CASE
    return fail(FCB_ENOTSUP, "point dimension must be 1, 2 or 3");
}

#ifndef FCB_RPT32
#define FCB_RPT32 3  // measured at config 4: 3 > 2 (+7 % solve), 4 spills or halves occupancy
#endif
constexpr int RPT_F32 = FCB_RPT32;  // rows per thread of the fp32 sweeps
constexpr int RPT_F64 = 1;

template <typename Real, int RPT>
static size_t ot_ws_bytes_t(int mode, int n, int m, int d) {
    int grid = 0;
    int rc = 0;
    if (d == 1) rc = ot_grid_size<Real, 1, RPT, true>(&grid);
    else if (d == 2) rc = ot_grid_size<Real, 2, RPT, true>(&grid);
    else rc = ot_grid_size<Real, 3, RPT, true>(&grid);
    if (rc) grid = 2 * sm_count();
    // the BARY=false instantiation may have a different occupancy: size for
    // the larger of the two possible grids
    int grid2 = 0;
    if (d == 1) rc = ot_grid_size<Real, 1, RPT, false>(&grid2);
    else if (d == 2) rc = ot_grid_size<Real, 2, RPT, false>(&grid2);
    else rc = ot_grid_size<Real, 3, RPT, false>(&grid2);
    if (rc) grid2 = grid;
    OtLayout<Real> L1, L2;
    ot_layout<Real>(L1, mode, n, m, d, RPT, grid, nullptr, 0);
    ot_layout<Real>(L2, mode, n, m, d, RPT, grid2, nullptr, 0);
    return std::max(L1.bytes, L2.bytes);
}

size_t ot_ws_bytes(int mode, int precision, int n, int m, int d) {
    if (d < 1 || d > 3) return 0;
    if (precision == FCB_FP64) return ot_ws_bytes_t<double, RPT_F64>(mode, n, m, d);
    return ot_ws_bytes_t<float, RPT_F32>(mode, n, m, d);
}

int ot_solve(int mode, int precision, const double* X, int n, const double* Y, int m, int d,
             const double* scal, int max_iters, double tol, const double* f0, double* f, double* g,
             double* rs, double* stat, double* bary, const int* gate, void* ws, size_t ws_bytes,
             cudaStream_t st) {
    if (n < 1 || (mode != FCB_OT_SYM && m < 1)) return fail(FCB_EINPUT, "empty point set");
    if (max_iters < 1) return fail(FCB_EINPUT, "max_iters must be >= 1");
    if (mode == FCB_OT_SWEEP && !f0) return fail(FCB_EINPUT, "sweep needs a potential");
    if (precision == FCB_FP64)
        return ot_dispatch<double, RPT_F64>(mode, d, X, n, Y, m, scal, max_iters, tol, f0, f, g, rs,
                                            stat, bary, gate, ws, ws_bytes, st);
    return ot_dispatch<float, RPT_F32>(mode, d, X, n, Y, m, scal, max_iters, tol, f0, f, g, rs,
                                       stat, bary, gate, ws, ws_bytes, st);
}

// One LSE sweep with an epilogue (M-sharded solves, distributed.py):
//   L_i = LSE_j((pot_j - |r_i - s_j|^2) / omega)            (sinkhorn.py:151-167)
//   out_i = scale omega (shift - L_i)  (scale != 0)   or   L_i
//   bary (nullable, nr x (d+1)): {L_i, softmax-weighted mean of the columns}
template <typename Real, int RPT>
static int lse_sweep_t(int d, const double* R, int nr, const double* S, int ns, const double* scal,
                       const double* pot, double* out, double* bary, const int* gate, void* ws,
                       size_t ws_bytes, cudaStream_t st, OtEpi epi) {
#define FCB_LS_CASE(DD)                                                                           \
    if (d == DD) {                                                                                \
        if (bary)                                                                                 \
            return ot_launch<Real, DD, RPT, true>(FCB_OT_SWEEP, R, nr, S, ns, scal, 1, 0.0, pot,   \
                                                  out, nullptr, nullptr, nullptr, bary, gate, ws, \
                                                  ws_bytes, st, epi);                             \
        return ot_launch<Real, DD, RPT, false>(FCB_OT_SWEEP, R, nr, S, ns, scal, 1, 0.0, pot, out, \
                                               nullptr, nullptr, nullptr, nullptr, gate, ws,      \
                                               ws_bytes, st, epi);                                \
    }
    FCB_LS_CASE(1)
    FCB_LS_CASE(2)
    FCB_LS_CASE(3)
#undef FCB_LS_CASE
    return fail(FCB_ENOTSUP, "point dimension must be 1, 2 or 3");
}

int lse_sweep(int precision, const double* R, int nr, const double* S, int ns, int d,
              const double* scal, const double* pot, const double* row_est, double row_logw,
              double out_scale, double out_shift, double* out, double* bary, const int* gate,
              void* ws, size_t ws_bytes, cudaStream_t st) {
    if (nr < 1 || ns < 1) return fail(FCB_EINPUT, "empty point set");
    if (!pot) return fail(FCB_EINPUT, "sweep needs a potential");
    OtEpi epi;
    epi.scale = out_scale;
    epi.shift = out_shift;
    epi.bary_L = 1;
    epi.row_est = row_est;
    epi.row_logw = row_logw;
    if (precision == FCB_FP64)
        return lse_sweep_t<double, RPT_F64>(d, R, nr, S, ns, scal, pot, out, bary, gate, ws,
                                            ws_bytes, st, epi);
    return lse_sweep_t<float, RPT_F32>(d, R, nr, S, ns, scal, pot, out, bary, gate, ws, ws_bytes,
                                       st, epi);
}

size_t omega_ws_bytes(int n, int m) {
    (void)n;
    (void)m;
    return 2 * ST_GRID * 4 * sizeof(double) + 512;
}

// Two launches: pair statistics, then omega/centring (+ optional self-term
// scal and warm-start selection for sinkhorn_flow).
static int omega_prep(int mode, const double* X, int n, const double* Y, int m, int d,
                      double omega_fixed, double unit, double* scal, double* scal_self,
                      const double* warm_f, const double* warm_p, const int* warm_valid,
                      double* f0, double* p0, unsigned* zero_count, void* ws, size_t ws_bytes,
                      cudaStream_t st) {
    if (ws_bytes < omega_ws_bytes(n, m)) return fail(FCB_EWORKSPACE, "omega workspace too small");
    double* part = static_cast<double*>(ws);
    const bool haveY = (mode == FCB_OT_ASYM || mode == FCB_OT_SWEEP) && Y != nullptr && m > 0;
    const int gx = stats_blocks(n);
    const int gy = haveY ? stats_blocks(m) : 0;
    pair_stats_kernel<<<gx + gy, ST_BLOCK, 0, st>>>(X, n, Y, m, d, gx, part);
    FCB_LAUNCHED("pair_stats_kernel");
    flow_prep_kernel<<<1, PREP_BLOCK, 0, st>>>(part, gx, gy, n, m, d, mode, omega_fixed, unit, scal,
                                               scal_self, warm_f, warm_p, warm_valid, f0, p0,
                                               zero_count);
    FCB_LAUNCHED("flow_prep_kernel");
    return FCB_OK;
}

int resolve_omega(int mode, const double* X, int n, const double* Y, int m, int d,
                  double omega_fixed, double unit, double* scal, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
    return omega_prep(mode, X, n, Y, m, d, omega_fixed, unit, scal, nullptr, nullptr, nullptr,
                      nullptr, nullptr, nullptr, nullptr, ws, ws_bytes, st);
}

// ---------------------------------------------------------------------------
// small epilogue kernels
// ---------------------------------------------------------------------------
__global__ void ot_cost_kernel(int mode, const double* __restrict__ f, const double* __restrict__ rs,
                               int n, const double* __restrict__ g, int m, double* out) {
    __shared__ double scratch[32];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < n; i += 1024) a += f[i] * rs[i];
    if (mode == FCB_OT_ASYM)
        for (int j = threadIdx.x; j < m; j += 1024) b += g[j];
    a = block_sum<1024>(a, scratch);
    b = block_sum<1024>(b, scratch);
    if (threadIdx.x == 0) *out = (mode == FCB_OT_ASYM) ? a + b / m : 2.0 * a;
}

__global__ void ot_plan_kernel(const double* __restrict__ X, int n, const double* __restrict__ Y,
                               int m, int d, const double* __restrict__ f,
                               const double* __restrict__ g, const double* __restrict__ scal,
                               double* __restrict__ out) {
    const double w = scal[SC_OMEGA];
    const size_t total = (size_t)n * m;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
         t += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(t / m), j = (int)(t % m);
        double c2 = 0.0;
        for (int k = 0; k < d; ++k) {
            double df = __dadd_rn(X[(size_t)i * d + k], -Y[(size_t)j * d + k]);
            c2 = __dadd_rn(c2, __dmul_rn(df, df));
        }
        out[t] = exp((f[i] + g[j] - c2) / w);
    }
}

// OT(Y, Y) cache of the divergence: Y is fixed for a whole
// plan, so when omega is too (a numeric SinkhornConfig.omega) the M x M self
// solve is run once.  cache (caller-owned double[5], zeroed = empty):
// {valid, omega, cost, m, hits}.  Check: the self-Y solve's gate is set on a
// hit (or when the caller's gate already stops everything); commit: a hit
// replaces the (skipped) solve's cost, a miss stores it.  The cost of a hit is
// the stored double, so cached and uncached divergences are bit-identical.
__global__ void yy_cache_check_kernel(const double* scal, const double* cache, int m,
                                      const int* gate, int* gate_yy) {
    if (threadIdx.x == 0) {
        const bool stop = gate && *((volatile const int*)gate) != 0;
        const bool hit = cache[0] == 1.0 && cache[1] == scal[SC_OMEGA] && cache[3] == (double)m;
        *gate_yy = (stop || hit) ? 1 : 0;
    }
}

__global__ void yy_cache_commit_kernel(const double* scal, double* cache, int m,
                                       const int* gate, double* cost_yy) {
    if (threadIdx.x == 0) {
        if (gate && *((volatile const int*)gate) != 0) return;
        const bool hit = cache[0] == 1.0 && cache[1] == scal[SC_OMEGA] && cache[3] == (double)m;
        if (hit) {
            *cost_yy = cache[2];
            cache[4] += 1.0;
        } else {
            cache[0] = 1.0;
            cache[1] = scal[SC_OMEGA];
            cache[2] = *cost_yy;
            cache[3] = (double)m;
        }
    }
}

__global__ void divergence_combine_kernel(const double* costs, double* out) {
    if (threadIdx.x == 0) {
        out[1] = costs[0];
        out[2] = costs[1];
        out[3] = costs[2];
        out[0] = costs[0] - 0.5 * (costs[1] + costs[2]);
    }
}

__global__ void copy_scal_kernel(const double* src, double* dst, const double* centre_from,
                                 int d) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < 16; ++k) dst[k] = src[k];
        for (int k = 0; k < 3; ++k) dst[SC_C + k] = (k < d) ? centre_from[k] : 0.0;
    }
}

// Workspace of sinkhorn_flow: scalars, both solves' outputs and their
// OT layouts (both live at once in the one-launch flow kernel).
struct FlowWs {
    double* scal;
    double* scal_self;
    double* part;
    double* fin_part;
    double *f, *g, *rs_x, *stat_x, *bary_x;
    double *p, *rs_p, *stat_p, *bary_p;
    char* ws_a;
    char* ws_b;
    size_t bytes_a, bytes_b;
    size_t total;
};

template <typename Real, int D, int RPT>
static int flow_grid_size(int* grid) {
    static int cached = -1;
    if (cached < 0) {
        int per_sm = 0;
        FCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flow_kernel<Real, D, RPT>,
                                                               OT_BLOCK, 0));
        if (per_sm < 1) return fail(FCB_ECUDA, "flow_kernel cannot be resident");
        int cap = 2;
        if (const char* env = getenv("FCB_OT_CTAS_PER_SM")) cap = std::max(1, atoi(env));
        cached = std::min(per_sm, cap) * sm_count();
    }
    *grid = cached;
    return FCB_OK;
}

template <typename Real>
static FlowWs flow_layout_t(int n, int m, int d, int rpt, int grid, void* ws, size_t bytes) {
    Arena ar(ws, bytes);
    FlowWs L{};
    L.scal = ar.take<double>(16);
    L.scal_self = ar.take<double>(16);
    L.part = ar.take<double>((size_t)grid * 8);
    L.fin_part = ar.take<double>(grid);
    L.f = ar.take<double>(n);
    L.g = ar.take<double>(m);
    L.rs_x = ar.take<double>(n);
    L.stat_x = ar.take<double>(4);
    L.bary_x = ar.take<double>((size_t)n * (d + 1));
    L.p = ar.take<double>(n);
    L.rs_p = ar.take<double>(n);
    L.stat_p = ar.take<double>(4);
    L.bary_p = ar.take<double>((size_t)n * (d + 1));
    OtLayout<Real> la, lb;
    ot_layout<Real>(la, FCB_OT_ASYM, n, m, d, rpt, grid, nullptr, 0);
    ot_layout<Real>(lb, FCB_OT_SYM, n, n, d, rpt, grid, nullptr, 0);
    L.bytes_a = la.bytes;
    L.bytes_b = lb.bytes;
    L.ws_a = ar.take<char>(la.bytes);
    L.ws_b = ar.take<char>(lb.bytes);
    L.total = ar.off + 256;
    return L;
}

template <typename Real, int RPT>
static int flow_grid_any(int d, int* grid) {
    if (d == 1) return flow_grid_size<Real, 1, RPT>(grid);
    if (d == 2) return flow_grid_size<Real, 2, RPT>(grid);
    return flow_grid_size<Real, 3, RPT>(grid);
}

// flow_resident.cu: the one-launch flow with the point sets in shared memory
bool sinkhorn_flow_resident_fits(int n, int m, int d);
size_t sinkhorn_flow_resident_ws_bytes(int n, int m, int d);
int sinkhorn_flow_resident(const double* X, int n, const double* Y, int m, int d,
                           double omega_fixed, int max_iters, double tol, double* warm_f,
                           double* warm_p, int* warm_valid, double* flow, double* fstat,
                           int* plan_state, int iteration, double* flow_log, double conv_tol,
                           void* ws, size_t ws_bytes, cudaStream_t st);

size_t sinkhorn_flow_ws_bytes(int precision, int n, int m, int d) {
    if (d < 1 || d > 3) return 0;
    if (precision != FCB_FP64 && sinkhorn_flow_resident_fits(n, m, d))
        return sinkhorn_flow_resident_ws_bytes(n, m, d);
    int grid = 0;
    if (precision == FCB_FP64) {
        if (flow_grid_any<double, RPT_F64>(d, &grid)) grid = 2 * sm_count();
        return flow_layout_t<double>(n, m, d, RPT_F64, grid, nullptr, 0).total;
    }
    if (flow_grid_any<float, RPT_F32>(d, &grid)) grid = 2 * sm_count();
    return flow_layout_t<float>(n, m, d, RPT_F32, grid, nullptr, 0).total;
}

static double unit_for(int precision) { return precision == FCB_FP64 ? 1.0 : kLog2e; }

template <typename Real, int D, int RPT>
static int flow_launch(const double* X, int n, const double* Y, int m, double omega_fixed,
                       int max_iters, double tol, double* warm_f, double* warm_p, int* warm_valid,
                       double* flow, double* fstat, int* plan_state, int iteration,
                       double* flow_log, double conv_tol, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
    int grid = 0;
    int rc = flow_grid_size<Real, D, RPT>(&grid);
    if (rc) return rc;
    FlowWs L = flow_layout_t<Real>(n, m, D, RPT, grid, ws, ws_bytes);
    if (L.total > ws_bytes) return fail(FCB_EWORKSPACE, "sinkhorn_flow workspace too small");
    FlowArgs<Real> fa{};
    OtLayout<Real> la, lb;
    ot_layout<Real>(la, FCB_OT_ASYM, n, m, D, RPT, grid, L.ws_a, L.bytes_a);
    ot_layout<Real>(lb, FCB_OT_SYM, n, n, D, RPT, grid, L.ws_b, L.bytes_b);
    fa.a = la.a;
    fa.b = lb.a;
    const double loga = -log((double)n), logb = -log((double)m);
    for (OtArgs<Real>* o : {&fa.a, &fa.b}) {
        o->X = X;
        o->max_iters = max_iters;
        o->tol = tol;
        o->loga = loga;
        o->bary = nullptr;
        o->gate = nullptr;
        o->scal = nullptr;
        o->f0 = nullptr;
    }
    fa.a.Y = Y;
    fa.a.logb = logb;
    fa.a.f_out = L.f;
    fa.a.g_out = L.g;
    fa.a.rs_out = L.rs_x;
    fa.a.stat = L.stat_x;
    fa.a.bary = L.bary_x;
    fa.b.Y = nullptr;
    fa.b.logb = 0.0;
    fa.b.f_out = L.p;
    fa.b.g_out = nullptr;
    fa.b.rs_out = L.rs_p;
    fa.b.stat = L.stat_p;
    fa.b.bary = L.bary_p;
    fa.b.bar = fa.a.bar;  // one barrier and work counter for the whole flow
    fa.omega_fixed = omega_fixed;
    fa.part = L.part;
    fa.scal = L.scal;
    fa.scal_self = L.scal_self;
    fa.warm_f = warm_f;
    fa.warm_p = warm_p;
    fa.warm_valid = (warm_f && warm_p) ? warm_valid : nullptr;
    fa.flow = flow;
    fa.fstat = fstat;
    fa.plan_state = plan_state;
    fa.iteration = iteration;
    fa.flow_log = flow_log;
    fa.conv_tol = conv_tol;
    fa.fin_part = L.fin_part;
    FCB_CUDA(cudaMemsetAsync(fa.a.bar, 0, sizeof(GridBarrier), st));
    void* args[] = {&fa};
    FCB_CUDA(cudaLaunchCooperativeKernel((const void*)flow_kernel<Real, D, RPT>, dim3(grid),
                                         dim3(OT_BLOCK), args, 0, st));
    FCB_LAUNCHED("flow_kernel");
    return FCB_OK;
}

int sinkhorn_flow(int precision, const double* X, int n, const double* Y, int m, int d,
                  double omega_fixed, int max_iters, double tol, double* warm_f, double* warm_p,
                  int* warm_valid, double* flow, double* fstat, int* plan_state, int iteration,
                  double* flow_log, double conv_tol, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
    if (n < 1 || m < 1) return fail(FCB_EINPUT, "empty point set");
    if (max_iters < 1) return fail(FCB_EINPUT, "max_iters must be >= 1");
    if (precision != FCB_FP64 && sinkhorn_flow_resident_fits(n, m, d))
        return sinkhorn_flow_resident(X, n, Y, m, d, omega_fixed, max_iters, tol, warm_f, warm_p,
                                      warm_valid, flow, fstat, plan_state, iteration, flow_log,
                                      conv_tol, ws, ws_bytes, st);
#define FCB_FLOW_CASE(DD)                                                                        \
    if (d == DD) {                                                                               \
        if (precision == FCB_FP64)                                                               \
            return flow_launch<double, DD, RPT_F64>(X, n, Y, m, omega_fixed, max_iters, tol,     \
                                                    warm_f, warm_p, warm_valid, flow, fstat,     \
                                                    plan_state, iteration, flow_log, conv_tol,   \
                                                    ws, ws_bytes, st);                           \
        return flow_launch<float, DD, RPT_F32>(X, n, Y, m, omega_fixed, max_iters, tol, warm_f,  \
                                               warm_p, warm_valid, flow, fstat, plan_state,      \
                                               iteration, flow_log, conv_tol, ws, ws_bytes, st); \
    }
    FCB_FLOW_CASE(1)
    FCB_FLOW_CASE(2)
    FCB_FLOW_CASE(3)
#undef FCB_FLOW_CASE
    return fail(FCB_ENOTSUP, "point dimension must be 1, 2 or 3");
}

struct DivWs {
    double* scal;
    void* omega_ws;
    double *f, *g, *rs, *stat, *costs;
    int* gate_yy;  // self-Y solve gate of the cached variant
    void* ot_ws;
    size_t ot_bytes, total;
};

static DivWs div_layout(int precision, int n, int m, int d, void* ws, size_t bytes) {
    Arena ar(ws, bytes);
    DivWs L{};
    const int nm = std::max(n, m);
    L.scal = ar.take<double>(16);
    L.omega_ws = ar.take<char>(omega_ws_bytes(n, m));
    L.f = ar.take<double>(nm);
    L.g = ar.take<double>(nm);
    L.rs = ar.take<double>(nm);
    L.stat = ar.take<double>(4);
    L.costs = ar.take<double>(4);
    L.gate_yy = ar.take<int>(4);
    L.ot_bytes = std::max(ot_ws_bytes(FCB_OT_ASYM, precision, n, m, d),
                          std::max(ot_ws_bytes(FCB_OT_SYM, precision, n, n, d),
                                   ot_ws_bytes(FCB_OT_SYM, precision, m, m, d)));
    L.ot_ws = ar.take<char>(L.ot_bytes);
    L.total = ar.off + 256;
    return L;
}

size_t sinkhorn_divergence_ws_bytes(int precision, int n, int m, int d) {
    return div_layout(precision, n, m, d, nullptr, 0).total;
}

int sinkhorn_divergence(int precision, const double* X, int n, const double* Y, int m, int d,
                        double omega_fixed, int max_iters, double tol, double* out,
                        const int* gate, void* ws, size_t ws_bytes, cudaStream_t st,
                        double* yy_cache) {
    DivWs L = div_layout(precision, n, m, d, ws, ws_bytes);
    if (L.total > ws_bytes) return fail(FCB_EWORKSPACE, "divergence workspace too small");
    int rc = resolve_omega(FCB_OT_ASYM, X, n, Y, m, d, omega_fixed, unit_for(precision), L.scal,
                           L.omega_ws, omega_ws_bytes(n, m), st);
    if (rc) return rc;
    rc = ot_solve(FCB_OT_ASYM, precision, X, n, Y, m, d, L.scal, max_iters, tol, nullptr, L.f, L.g,
                  L.rs, L.stat, nullptr, gate, L.ot_ws, L.ot_bytes, st);
    if (rc) return rc;
    ot_cost_kernel<<<1, 1024, 0, st>>>(FCB_OT_ASYM, L.f, L.rs, n, L.g, m, L.costs + 0);
    FCB_LAUNCHED("ot_cost_kernel");
    // self terms: same omega, centre on the set itself
    copy_scal_kernel<<<1, 32, 0, st>>>(L.scal, L.scal, L.scal + SC_MX, d);
    FCB_LAUNCHED("copy_scal_kernel");
    rc = ot_solve(FCB_OT_SYM, precision, X, n, nullptr, 0, d, L.scal, max_iters, tol, nullptr, L.f,
                  nullptr, L.rs, L.stat, nullptr, gate, L.ot_ws, L.ot_bytes, st);
    if (rc) return rc;
    ot_cost_kernel<<<1, 1024, 0, st>>>(FCB_OT_SYM, L.f, L.rs, n, nullptr, 0, L.costs + 1);
    FCB_LAUNCHED("ot_cost_kernel");
    copy_scal_kernel<<<1, 32, 0, st>>>(L.scal, L.scal, L.scal + SC_MY, d);
    FCB_LAUNCHED("copy_scal_kernel");
    const int* gate_yy = gate;
    if (yy_cache) {
        yy_cache_check_kernel<<<1, 32, 0, st>>>(L.scal, yy_cache, m, gate, L.gate_yy);
        FCB_LAUNCHED("yy_cache_check_kernel");
        gate_yy = L.gate_yy;
    }
    rc = ot_solve(FCB_OT_SYM, precision, Y, m, nullptr, 0, d, L.scal, max_iters, tol, nullptr, L.f,
                  nullptr, L.rs, L.stat, nullptr, gate_yy, L.ot_ws, L.ot_bytes, st);
    if (rc) return rc;
    ot_cost_kernel<<<1, 1024, 0, st>>>(FCB_OT_SYM, L.f, L.rs, m, nullptr, 0, L.costs + 2);
    FCB_LAUNCHED("ot_cost_kernel");
    if (yy_cache) {
        yy_cache_commit_kernel<<<1, 32, 0, st>>>(L.scal, yy_cache, m, gate, L.costs + 2);
        FCB_LAUNCHED("yy_cache_commit_kernel");
    }
    divergence_combine_kernel<<<1, 32, 0, st>>>(L.costs, out);
    FCB_LAUNCHED("divergence_combine_kernel");
    return FCB_OK;
}

int ot_cost(int mode, const double* f, const double* rs, int n, const double* g, int m,
            double* out, cudaStream_t st) {
    ot_cost_kernel<<<1, 1024, 0, st>>>(mode, f, rs, n, g, m, out);
    FCB_LAUNCHED("ot_cost_kernel");
    return FCB_OK;
}

int ot_plan(const double* X, int n, const double* Y, int m, int d, const double* f,
            const double* g, const double* scal, double* out, cudaStream_t st) {
    const size_t total = (size_t)n * m;
    const int blocks = (int)std::min<size_t>(148 * 8, (total + 255) / 256);
    ot_plan_kernel<<<std::max(blocks, 1), 256, 0, st>>>(X, n, Y, m, d, f, g, scal, out);
    FCB_LAUNCHED("ot_plan_kernel");
    return FCB_OK;
}

}  // namespace fcb

// Debug: copy the grid-barrier timeline of FCB_TIMELINE builds (host array of
// up to `cap` ns timestamps, two per barrier: arrival and release of block 0)
// and reset it.  Returns the count (always 0 in production builds).
extern "C" FCB_API int fcb_debug_timeline(unsigned long long* host_out, int cap) {
#ifdef FCB_TIMELINE
    unsigned n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, fcb::g_timeline_n, sizeof(unsigned));
    n = n > 8192u ? 8192u : n;
    const unsigned k = (unsigned)cap < n ? (unsigned)cap : n;
    if (k) cudaMemcpyFromSymbol(host_out, fcb::g_timeline, k * sizeof(unsigned long long));
    unsigned zero = 0;
    cudaMemcpyToSymbol(fcb::g_timeline_n, &zero, sizeof(unsigned));
    return (int)k;
#else
    (void)host_out;
    (void)cap;
    return 0;
#endif
}

extern "C" FCB_API long long fcb_debug_careful_items(void) {
    unsigned v = 0, zero = 0;
    if (cudaMemcpyFromSymbol(&v, fcb::g_careful_items, sizeof(unsigned)) != cudaSuccess) return -1;
    cudaMemcpyToSymbol(fcb::g_careful_items, &zero, sizeof(unsigned));
    return (long long)v;
}
