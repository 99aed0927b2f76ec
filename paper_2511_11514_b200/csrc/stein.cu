// stein.cu -- density score, median bandwidth and the Stein variational flow.
//
// Replaces reference.py:77-110 (GaussianMixture._component_terms / score /
// log_density) and stein.py:66-140 (median_bandwidth, stein_flow).
//
// * gmm_eval: one thread per point, fp64, K components streamed with an
//   online-softmax over the responsibilities (coalesced point I/O).
// * median: the reference takes np.median over all n^2 pairwise distances
//   (diagonal zeros included; stein.py:75).  Here the exact order statistics
//   are found by a 6-pass radix select over the float64 bit patterns of the
//   squared distances (11-bit digits, histograms in shared memory), never
//   storing the n^2 matrix.  Squared distances are formed with the same
//   operation order as _pairwise_sq (stein.py:57-63) and without FMA
//   contraction, so the selected values are bit-identical to numpy's.
// * stein_flow: g_i = (1/n)[sum_j k_ij w_j + (2/h) x'_i sum_j k_ij],
//   w_j = s_j - (2/h) x'_j, k_ij = exp(-|x_i-x_j|^2/h), fused in registers
//   over column chunks with a fixed-order merge (no float atomics).
#include <cstddef>

#include "fcb_internal.cuh"
#include "stein_dev.cuh"

#include <cooperative_groups.h>
#include <mutex>

#include <algorithm>

namespace fcb {

// ---------------------------------------------------------------------------
// Gaussian mixture score / log density
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) gmm_eval_kernel(const double* __restrict__ X, int n, int k,
                                                       const double* __restrict__ prm,
                                                       double* __restrict__ score,
                                                       double* __restrict__ logdens,
                                                       const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        gmm_point<D>(X + (size_t)i * D, k, prm, score ? score + (size_t)i * D : nullptr,
                     logdens ? logdens + i : nullptr);
}

// SamplePoints.sample (reference.py:140-146) on a device-resident cloud: the
// indices are drawn on the host (numpy PCG64, bit-identical to the
// reference) and the rows are gathered here, one thread per output element
// so consecutive threads write consecutive doubles.  An out-of-range index
// stores its position in *status (first one wins) and the row is left zero.
__global__ void gather_rows_kernel(const double* __restrict__ src, int m, int d,
                                   const int* __restrict__ idx, int n, double* __restrict__ out,
                                   int* status) {
    const size_t total = (size_t)n * d;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
        const size_t i = e / d, q = e % d;
        const int j = __ldg(idx + i);
        if (j < 0 || j >= m) {
            out[e] = 0.0;
            if (q == 0 && status) atomicCAS(status, -1, (int)i);
            continue;
        }
        out[e] = __ldg(src + (size_t)j * d + q);
    }
}

int gather_rows(const double* src, int m, int d, const int* idx, int n, double* out, int* status,
                cudaStream_t st) {
    if (n < 1) return FCB_OK;
    if (m < 1 || d < 1) return fail(FCB_EINPUT, "gather: empty source");
    if (status) FCB_CUDA(cudaMemsetAsync(status, 0xff, sizeof(int), st));
    const long total = (long)n * d;
    const int blocks = (int)std::max<long>(1, std::min<long>(8L * sm_count(), (total + 255) / 256));
    gather_rows_kernel<<<blocks, 256, 0, st>>>(src, m, d, idx, n, out, status);
    FCB_LAUNCHED("gather_rows_kernel");
    return FCB_OK;
}

int gmm_eval(const double* X, int n, int d, int k, const double* prm, double* score,
             double* logdens, const int* gate, cudaStream_t st) {
    if (n < 1) return FCB_OK;
    const int blocks = std::min(4 * sm_count(), (n + 255) / 256);
    switch (d) {
        case 1: gmm_eval_kernel<1><<<blocks, 256, 0, st>>>(X, n, k, prm, score, logdens, gate); break;
        case 2: gmm_eval_kernel<2><<<blocks, 256, 0, st>>>(X, n, k, prm, score, logdens, gate); break;
        case 3: gmm_eval_kernel<3><<<blocks, 256, 0, st>>>(X, n, k, prm, score, logdens, gate); break;
        default: return fail(FCB_ENOTSUP, "gmm dimension must be 1, 2 or 3");
    }
    FCB_LAUNCHED("gmm_eval_kernel");
    return FCB_OK;
}

// ---------------------------------------------------------------------------
// exact median of the n^2 pairwise distances (radix select)
// ---------------------------------------------------------------------------
constexpr int MED_TILE = 64;
constexpr int MED_BLOCK = 256;
constexpr int MED_BINS = 2048;
constexpr int MED_PASSES = 6;
constexpr long long MED_COOP_TILES = 16384;  // one cooperative launch up to n ~ 11.5k
__constant__ int c_med_shift[MED_PASSES] = {52, 41, 30, 19, 8, 0};
__constant__ int c_med_bits[MED_PASSES] = {11, 11, 11, 11, 11, 8};

struct MedState {
    unsigned long long prefix[2];  // selected high bits so far (lo, hi target)
    unsigned long long rank[2];    // remaining rank inside the prefix bucket
    unsigned long long hist[2][MED_BINS];
    unsigned done;                 // CTAs finished with the current pass
    GridBarrier bar;               // median_coop_kernel
};

// The digit selection of one radix pass, by one CTA of MED_BLOCK threads:
// each thread owns MED_BINS / MED_BLOCK consecutive bins, a block-wide
// exclusive scan of the per-thread counts locates the bin holding each target
// rank.  Then the histograms are cleared for the next pass.
__device__ void median_select_block(MedState* st, int n, int pass) {
    constexpr int PER = MED_BINS / MED_BLOCK;
    __shared__ unsigned long long s_warp[MED_BLOCK / 32];
    __shared__ unsigned long long s_new[2][2];  // {prefix, rank} per target
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int bits = c_med_bits[pass];
    const int nbins = 1 << bits;
    const unsigned long long p0 = st->prefix[0], p1 = st->prefix[1];
    const bool same = p0 == p1;
    for (int t = 0; t < 2; ++t) {
        const unsigned long long* h = st->hist[same ? 0 : t];
        const unsigned long long pre = t ? p1 : p0;
        // the n diagonal zeros live in bucket 0 while the prefix is 0
        const unsigned long long zeros = (pre == 0ull) ? (unsigned long long)n : 0ull;
        unsigned long long c[PER], sum = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int b = tid * PER + k;
            c[k] = (b < nbins) ? __ldcg(h + b) + (b == 0 ? zeros : 0ull) : 0ull;
            sum += c[k];
        }
        unsigned long long incl = sum;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        unsigned long long base = 0;
        for (int w = 0; w < wid; ++w) base += s_warp[w];
        const unsigned long long excl = base + incl - sum;
        const unsigned long long r = st->rank[t];
        const bool last = tid == MED_BLOCK - 1;
        if ((r >= excl && r < excl + sum) || (last && r >= excl + sum)) {
            unsigned long long rr = r - excl;
            int b = tid * PER;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                if (rr < c[k] || k == PER - 1) break;
                rr -= c[k];
                ++b;
            }
            b = min(b, nbins - 1);  // past the end only for inconsistent counts
            s_new[t][0] = (pre << bits) | (unsigned long long)b;
            s_new[t][1] = rr;
        }
        __syncthreads();
    }
    if (tid == 0) {
        st->prefix[0] = s_new[0][0];
        st->rank[0] = s_new[0][1];
        st->prefix[1] = s_new[1][0];
        st->rank[1] = s_new[1][1];
        st->done = 0u;
    }
    for (int b = tid; b < 2 * MED_BINS; b += MED_BLOCK) (&st->hist[0][0])[b] = 0ull;
}


// One radix pass over tiles [t_lo, t_hi) of the upper triangle of 64 x 64
// pair tiles (tile t handled by CTA t % gridDim.x): shared-memory histograms
// of the current digit among keys that match the known prefix, then one
// global atomic per nonzero bin.
template <int D>
__device__ __forceinline__ void median_hist_pass(const double* __restrict__ X, int n, MedState* st,
                                                 int pass, long long t_lo, long long t_hi,
                                                 unsigned (*hist)[MED_BINS], double* pj) {
    const int shift = c_med_shift[pass];
    const int bits = c_med_bits[pass];
    const int hshift = shift + bits;  // bits above the current digit are known
    const unsigned long long pre0 = __ldcg(&st->prefix[0]), pre1 = __ldcg(&st->prefix[1]);
    const bool same = pre0 == pre1;
    for (int b = threadIdx.x; b < 2 * MED_BINS; b += MED_BLOCK) (&hist[0][0])[b] = 0u;
    const int nb = (n + MED_TILE - 1) / MED_TILE;
    __syncthreads();
    for (long long t = t_lo + blockIdx.x; t < t_hi; t += gridDim.x) {
        // map t -> (bi, bj) with bi <= bj (row-major upper triangle)
        int bi = (int)((2.0 * nb + 1.0 - sqrt((2.0 * nb + 1.0) * (2.0 * nb + 1.0) - 8.0 * t)) / 2.0);
        bi = max(0, min(bi, nb - 1));
        while (bi > 0 && (long long)bi * nb - (long long)bi * (bi - 1) / 2 > t) --bi;
        while ((long long)(bi + 1) * nb - (long long)(bi + 1) * bi / 2 <= t) ++bi;
        const long long row_start = (long long)bi * nb - (long long)bi * (bi - 1) / 2;
        const int bj = bi + (int)(t - row_start);
        __syncthreads();
        for (int k = threadIdx.x; k < MED_TILE * D; k += MED_BLOCK) {
            const int j = bj * MED_TILE + k / D;
            pj[k] = (j < n) ? X[(size_t)j * D + (k % D)] : 0.0;
        }
        __syncthreads();
        // each thread: one i row (64 rows / 4 threads per row) x 16 columns
        const int il = threadIdx.x >> 2;
        const int jq = threadIdx.x & 3;
        const int i = bi * MED_TILE + il;
        if (i < n) {
            double xi[D];
#pragma unroll
            for (int q = 0; q < D; ++q) xi[q] = X[(size_t)i * D + q];
            for (int jj = jq; jj < MED_TILE; jj += 4) {
                const int j = bj * MED_TILE + jj;
                if (j >= n || j <= i) continue;
                const unsigned long long key = sqdist_key<D>(xi, &pj[jj * D]);
                const unsigned long long hi = (hshift >= 64) ? 0ull : (key >> hshift);
                const unsigned dig = (unsigned)((key >> shift) & ((1ull << bits) - 1ull));
                if (hi == pre0) atomicAdd(&hist[0][dig], 2u);
                if (!same && hi == pre1) atomicAdd(&hist[1][dig], 2u);
            }
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < MED_BINS; b += MED_BLOCK) {
        if (hist[0][b]) atomicAdd(&st->hist[0][b], (unsigned long long)hist[0][b]);
        if (!same && hist[1][b]) atomicAdd(&st->hist[1][b], (unsigned long long)hist[1][b]);
    }
}

// Tiles [t_lo, t_hi) of the upper triangle of 64 x 64 pair tiles.  fold: the
// last CTA selects the digit (single GPU); 0 leaves the histogram for an
// all_reduce across ranks and fcb_median_select (M-sharded median).
template <int D>
__global__ void __launch_bounds__(MED_BLOCK) median_hist_kernel(const double* __restrict__ X, int n,
                                                                MedState* st, int pass,
                                                                const int* gate, long long t_lo,
                                                                long long t_hi, int fold) {
    __shared__ unsigned hist[2][MED_BINS];
    __shared__ double pj[MED_TILE * D];
    if (gate && *((volatile const int*)gate) != 0) return;
    median_hist_pass<D>(X, n, st, pass, t_lo, t_hi, hist, pj);
    if (!fold) return;
    // the last CTA of the pass selects the digit (no separate launch)
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&st->done, 1u) == gridDim.x - 1) ? 1 : 0;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    median_select_block(st, n, pass);
}

__global__ void median_init_kernel(MedState* st, unsigned long long klo, unsigned long long khi,
                                   const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    for (int b = threadIdx.x; b < 2 * MED_BINS; b += blockDim.x) (&st->hist[0][0])[b] = 0ull;
    if (threadIdx.x == 0) {
        st->prefix[0] = st->prefix[1] = 0ull;
        st->rank[0] = klo;
        st->rank[1] = khi;
        st->done = 0u;
    }
}

// the selected pair -> hstat (median_finish_vals, stein_dev.cuh)
__device__ __forceinline__ void median_finish_dev(const MedState* st, int n, double log_np1,
                                                  double* hstat) {
    median_finish_vals(__ldcg(&st->prefix[0]), __ldcg(&st->prefix[1]), n, log_np1, hstat);
}

// ---------------------------------------------------------------------------
// Small point sets (config 1: n = 500, 124750 pairs): ONE thread-block
// cluster.  The CTAs split the upper-triangle pairs, compute each distance key
// once into shared memory (pass 0) and re-scan their keys in the later passes;
// per pass the histograms are merged over distributed shared memory (each CTA
// sums a slice of the bins of every CTA into CTA 0) and CTA 0 selects the
// digit.  Three cluster barriers per pass instead of two grid barriers through
// global memory and no global atomics (the cooperative kernel spends ~9 us per
// pass at n = 500 on 36 CTAs).
// ---------------------------------------------------------------------------
constexpr int MCL_BLOCK = 1024;
constexpr int MCL_SLICE = 2 * MED_BINS;  // bins of both targets

struct MclShared {
    unsigned long long pre[2], rank[2];  // identical in every CTA
    unsigned long long warp[2 * (MCL_BLOCK / 32)];
    unsigned long long wbase[2][MCL_BLOCK / 32];
    unsigned long long nw[2][3];
    unsigned long long bcnt[2];  // count of the selected bin (pairs x2, zeros included)
    unsigned ncand;              // CTA 0: candidates gathered for the final select
};
constexpr int MCL_CAND = 1024;  // candidate cap of the final O(m^2) rank select

inline size_t mcl_smem_bytes(int n, int d, long long keys_per_cta) {
    return align_up((size_t)n * d * sizeof(double), 16) + (size_t)keys_per_cta * 8 +
           2 * (size_t)MCL_SLICE * sizeof(unsigned);
}

// digit selection over the merged (2 x MED_BINS) counts (both targets at
// once; warp totals scanned by one warp), run by every CTA on its own copy of
// the merged histogram.
__device__ void mcl_select(const unsigned* merged, int n, int pass, MclShared& sh) {
    constexpr int PER = MED_BINS / MCL_BLOCK;
    constexpr int NW = MCL_BLOCK / 32;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int bits = c_med_bits[pass];
    const int nbins = 1 << bits;
    const unsigned long long p0 = sh.pre[0], p1 = sh.pre[1];
    const bool same = p0 == p1;
    unsigned long long c[2][PER], sum[2], incl[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const unsigned* h = merged + (same ? 0 : t) * MED_BINS;
        const unsigned long long zeros = ((t ? p1 : p0) == 0ull) ? (unsigned long long)n : 0ull;
        sum[t] = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int b = tid * PER + k;
            c[t][k] = (b < nbins) ? (unsigned long long)h[b] + (b == 0 ? zeros : 0ull) : 0ull;
            sum[t] += c[t][k];
        }
        incl[t] = sum[t];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long v = __shfl_up_sync(0xffffffffu, incl[t], o);
            if (lane >= o) incl[t] += v;
        }
        if (lane == 31) sh.warp[t * NW + wid] = incl[t];
    }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the warp totals, both targets
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const unsigned long long w = sh.warp[t * NW + lane];
            unsigned long long x = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long v = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += v;
            }
            sh.wbase[t][lane] = x - w;
        }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const unsigned long long excl = sh.wbase[t][wid] + incl[t] - sum[t];
        const unsigned long long r = sh.rank[t];
        const bool last = tid == MCL_BLOCK - 1;
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
            sh.nw[t][0] = ((t ? p1 : p0) << bits) | (unsigned long long)b;
            sh.nw[t][1] = rr;
            sh.nw[t][2] = cb;
        }
    }
    __syncthreads();
    if (tid == 0) {
        sh.pre[0] = sh.nw[0][0];
        sh.rank[0] = sh.nw[0][1];
        sh.bcnt[0] = sh.nw[0][2];
        sh.pre[1] = sh.nw[1][0];
        sh.rank[1] = sh.nw[1][1];
        sh.bcnt[1] = sh.nw[1][2];
    }
    __syncthreads();
}

// Final select among the gathered candidates (CTA 0): the multiset of bucket
// t is z zeros (the diagonal, while the prefix is 0) followed by every
// candidate twice (pairs i<j stand for (i,j) and (j,i)); the key at the
// remaining rank is the candidate with 2 less <= r < 2 (less + eq).
__device__ void mcl_resolve(const unsigned long long* cand, int m, int kshift, int n,
                            MclShared& sh) {
    __shared__ unsigned long long s_res[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const unsigned long long pre = sh.pre[t];
        const unsigned long long z = (pre == 0ull) ? (unsigned long long)n : 0ull;
        const unsigned long long rr = sh.rank[t];
        if (threadIdx.x == 0 && rr < z) s_res[t] = 0ull;
        if (rr >= z) {
            const unsigned long long r = rr - z;
            for (int i = threadIdx.x; i < m; i += MCL_BLOCK) {
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
        sh.pre[0] = s_res[0];
        sh.pre[1] = s_res[1];
    }
    __syncthreads();
}

#ifdef MCL_TL
__device__ unsigned long long g_mcl_tl[2][64];
#define MCL_MARK(slot)                                                               \
    do {                                                                             \
        if (threadIdx.x == 0 && (rank == 0 || rank == NCT - 1)) {                    \
            unsigned long long t_;                                                   \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
            g_mcl_tl[rank == 0 ? 0 : 1][slot] = t_;                                  \
        }                                                                            \
    } while (0)
#else
#define MCL_MARK(slot) \
    do {               \
    } while (0)
#endif
template <int D, int NCT>
__global__ void __launch_bounds__(MCL_BLOCK)
    median_cluster_kernel(const double* __restrict__ X, int n, long long keys_per_cta,
                          unsigned long long klo, unsigned long long khi, double log_np1,
                          double* hstat, const int* gate) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char mcl_smem[];
    __shared__ MclShared sh;
    if (gate && *((volatile const int*)gate) != 0) return;  // uniform over the cluster
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x;
    double* xs = reinterpret_cast<double*>(mcl_smem);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(
        mcl_smem + (((size_t)n * D * sizeof(double) + 15) & ~(size_t)15));
    unsigned* hist = reinterpret_cast<unsigned*>(keys + keys_per_cta);  // 2 x MED_BINS
    unsigned* merged = hist + MCL_SLICE;                                 // CTA 0: 2 x MED_BINS
    MCL_MARK(0);
    for (int k = tid; k < n * D; k += MCL_BLOCK) xs[k] = X[k];
    if (tid == 0) {
        sh.pre[0] = sh.pre[1] = 0ull;
        sh.rank[0] = klo;
        sh.rank[1] = khi;
        sh.ncand = 0u;
    }
    __syncthreads();
    // this CTA's run [p0, p1) of the row-major upper-triangle pairs (i < j)
    const long long P = (long long)n * (n - 1) / 2;
    const long long p0 = P * rank / NCT, p1 = P * (rank + 1) / NCT;
    const int cnt = (int)(p1 - p0);
    MCL_MARK(42);
    {
        // pairs i < j folded into an H x W rectangle: rectangle row r holds
        // triangle row r (n-1-r pairs) followed by its partner row, so a pair
        // index needs one division instead of a square root (the key pass is
        // issue-bound on the cluster's 16 SMs)
        const bool even = (n & 1) == 0;
        const int W = even ? n - 1 : n;
        const float invW = 1.0f / (float)W;
        for (int k = tid; k < cnt; k += MCL_BLOCK) {
            const int q = (int)(p0 + k);
            int r = (int)((float)q * invW);
            if (r * W > q) --r;
            else if ((r + 1) * W <= q) ++r;
            const int c = q - r * W;
            const int len = n - 1 - r;
            int i, j;
            if (c < len) {
                i = r;
                j = r + 1 + c;
            } else {
                i = even ? n - 1 - r : n - 2 - r;
                j = i + 1 + (c - len);
            }
            keys[k] = sqdist_key<D>(xs + (size_t)i * D, xs + (size_t)j * D);
        }
    }
    for (int pass = 0; pass < MED_PASSES; ++pass) {
        MCL_MARK(1 + 6 * pass);
        const int shift = c_med_shift[pass];
        const int bits = c_med_bits[pass];
        const int hshift = shift + bits;
        const unsigned long long pre0 = sh.pre[0], pre1 = sh.pre[1];
        const bool same = pre0 == pre1;
        for (int b = tid; b < MCL_SLICE; b += MCL_BLOCK) hist[b] = 0u;
        __syncthreads();
        for (int k = tid; k < cnt; k += MCL_BLOCK) {
            const unsigned long long key = keys[k];
            const unsigned long long hi = (hshift >= 64) ? 0ull : (key >> hshift);
            const unsigned dig = (unsigned)((key >> shift) & ((1ull << bits) - 1ull));
            if (hi == pre0) atomicAdd(&hist[dig], 2u);
            if (!same && hi == pre1) atomicAdd(&hist[MED_BINS + dig], 2u);
        }
        __syncthreads();
        MCL_MARK(2 + 6 * pass);
        cluster.sync();  // every CTA's histogram complete
        MCL_MARK(3 + 6 * pass);
        {
            // slice `rank` of the bins, summed over the cluster, written into
            // EVERY CTA's merged histogram (the stores spread over all the
            // receivers' shared-memory ports; one CTA reading for everyone
            // would serialise on its port)
            constexpr int PERB = MCL_SLICE / NCT;
            if (tid < PERB) {
                const int b = rank * PERB + tid;
                unsigned v[NCT];
#pragma unroll
                for (int r = 0; r < NCT; ++r) v[r] = *cluster.map_shared_rank(hist + b, r);
                unsigned acc = 0;
#pragma unroll
                for (int r = 0; r < NCT; ++r) acc += v[r];
#pragma unroll
                for (int r = 0; r < NCT; ++r) *cluster.map_shared_rank(merged + b, r) = acc;
            }
        }
        MCL_MARK(4 + 6 * pass);
        cluster.sync();  // merged histogram complete in every CTA
        MCL_MARK(5 + 6 * pass);
        mcl_select(merged, n, pass, sh);  // identical inputs -> identical prefixes
        MCL_MARK(6 + 6 * pass);
        // few keys left in the selected bucket(s): gather them into CTA 0 and
        // select exactly there instead of running the remaining passes
        const int kshift = shift;  // bits >= shift of the answers are known now
        if (pass + 1 < MED_PASSES) {
            unsigned long long m = 0;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                if (t == 1 && sh.pre[1] == sh.pre[0]) break;
                const unsigned long long z = (sh.pre[t] == 0ull) ? (unsigned long long)n : 0ull;
                m += (sh.bcnt[t] - min(z, sh.bcnt[t])) / 2ull;
            }
            if (m <= (unsigned long long)MCL_CAND) {  // uniform over the cluster
                unsigned long long* cand0 =
                    reinterpret_cast<unsigned long long*>(cluster.map_shared_rank(hist, 0));
                unsigned* nc0 = cluster.map_shared_rank(&sh.ncand, 0);
                const unsigned long long q0 = sh.pre[0], q1 = sh.pre[1];
                for (int k = tid; k < cnt; k += MCL_BLOCK) {
                    const unsigned long long key = keys[k];
                    const unsigned long long hi = key >> kshift;
                    if (hi == q0 || hi == q1) {
                        const unsigned slot = atomicAdd(nc0, 1u);
                        if (slot < (unsigned)MCL_CAND) cand0[slot] = key;
                    }
                }
                cluster.sync();  // candidates complete in CTA 0
                if (rank == 0)
                    mcl_resolve(reinterpret_cast<const unsigned long long*>(hist),
                                (int)min(sh.ncand, (unsigned)MCL_CAND), kshift, n, sh);
                break;
            }
        }
    }
    MCL_MARK(40);
    cluster.sync();  // no CTA exits while others may still read its shared memory
    MCL_MARK(41);
    if (rank == 0 && tid == 0) median_finish_vals(sh.pre[0], sh.pre[1], n, log_np1, hstat);
}

__global__ void median_finish_kernel(const MedState* st, int n, double log_np1, double* hstat,
                                     const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    if (threadIdx.x != 0) return;
    median_finish_dev(st, n, log_np1, hstat);
}

// Small and mid-size point sets (config 1: n = 500, 36 tiles): the whole
// selection in ONE cooperative launch -- init, then per radix pass the
// histogram over the CTAs' tiles, a grid barrier, the digit selection by
// CTA 0, a grid barrier -- instead of eight launches (at n = 500 each pass
// launch costs ~12 us of launch latency and tail for ~1 us of work).
template <int D>
__global__ void __launch_bounds__(MED_BLOCK)
    median_coop_kernel(const double* __restrict__ X, int n, MedState* st, long long ntiles,
                       unsigned long long klo, unsigned long long khi, double log_np1,
                       double* hstat, const int* gate) {
    __shared__ unsigned hist[2][MED_BINS];
    __shared__ double pj[MED_TILE * D];
    if (gate && *((volatile const int*)gate) != 0) return;
    if (blockIdx.x == 0) {
        for (int b = threadIdx.x; b < 2 * MED_BINS; b += MED_BLOCK) (&st->hist[0][0])[b] = 0ull;
        if (threadIdx.x == 0) {
            st->prefix[0] = st->prefix[1] = 0ull;
            st->rank[0] = klo;
            st->rank[1] = khi;
            st->done = 0u;
        }
    }
    grid_sync(&st->bar);
    for (int pass = 0; pass < MED_PASSES; ++pass) {
        median_hist_pass<D>(X, n, st, pass, 0, ntiles, hist, pj);
        grid_sync(&st->bar);
        if (blockIdx.x == 0) median_select_block(st, n, pass);
        grid_sync(&st->bar);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) median_finish_dev(st, n, log_np1, hstat);
}

__global__ void fixed_bandwidth_kernel(double h, double* hstat, const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    if (threadIdx.x == 0) {
        const bool clamped = h <= BANDWIDTH_FLOOR;
        hstat[0] = clamped ? BANDWIDTH_FLOOR : h;
        hstat[1] = NAN;
        hstat[2] = clamped ? 1.0 : 0.0;
        hstat[3] = 0.0;
    }
}

// One cluster of 16 CTAs (8 where 16 is not schedulable) when every CTA's keys
// fit in shared memory; FCB_ENOTSUP otherwise (the caller falls back to the
// cooperative / multi-launch selection).
#ifndef FCB_MED_CLUSTER
#define FCB_MED_CLUSTER 1
#endif
template <int D, int NCT>
static cudaError_t mcl_launch(const cudaLaunchConfig_t& cfg, const double* X, int n, long long per,
                              unsigned long long klo, unsigned long long khi, double log_np1,
                              double* hstat, const int* gate) {
    return cudaLaunchKernelEx(&cfg, median_cluster_kernel<D, NCT>, X, n, per, klo, khi, log_np1,
                              hstat, gate);
}

template <int NCT>
static const void* mcl_kernel(int d) {
    return d == 1 ? (const void*)median_cluster_kernel<1, NCT>
         : d == 2 ? (const void*)median_cluster_kernel<2, NCT>
                  : (const void*)median_cluster_kernel<3, NCT>;
}

static int median_cluster_launch(const double* X, int n, int d, double log_np1, double* hstat,
                                 const int* gate, cudaStream_t st) {
    if (!FCB_MED_CLUSTER || d < 1 || d > 3 || n < 2) return FCB_ENOTSUP;
    const long long P = (long long)n * (n - 1) / 2;
    // the one-time attribute setup below is shared by all host threads
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    static int max_smem = -1;
    if (max_smem < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) !=
            cudaSuccess)
            max_smem = 0;
    }
    // per (d, cluster size): the dynamic shared memory already granted, and
    // whether the cluster is schedulable at all (host calls cost ~us each and
    // this runs once per Stein iteration)
    static size_t granted[4][2] = {};
    static int usable[4][2] = {};  // 0 unknown, 1 yes, -1 no
    for (int nct : {16, 8}) {
        const int ci = nct == 16 ? 0 : 1;
        const long long per = (P + nct - 1) / nct;
        const size_t smem = mcl_smem_bytes(n, d, per);
        if (smem + sizeof(MclShared) + 1024 > (size_t)max_smem || usable[d][ci] < 0) continue;
        const void* kern = nct == 16 ? mcl_kernel<16>(d) : mcl_kernel<8>(d);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nct);
        cfg.blockDim = dim3(MCL_BLOCK);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = nct;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (smem > granted[d][ci]) {
            if ((nct > 8 && cudaFuncSetAttribute(
                                kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                                cudaSuccess) ||
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem) != cudaSuccess) {
                cudaGetLastError();
                usable[d][ci] = -1;
                continue;
            }
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess ||
                clusters < 1) {
                cudaGetLastError();
                continue;  // not at this size (larger smem); smaller sets may still fit
            }
            granted[d][ci] = smem;
            usable[d][ci] = 1;
        }
        const unsigned long long N = (unsigned long long)n * (unsigned long long)n;
        const unsigned long long klo = (N - 1ull) / 2ull, khi = N / 2ull;
        cudaError_t e;
        if (nct == 16) {
            e = d == 1 ? mcl_launch<1, 16>(cfg, X, n, per, klo, khi, log_np1, hstat, gate)
              : d == 2 ? mcl_launch<2, 16>(cfg, X, n, per, klo, khi, log_np1, hstat, gate)
                       : mcl_launch<3, 16>(cfg, X, n, per, klo, khi, log_np1, hstat, gate);
        } else {
            e = d == 1 ? mcl_launch<1, 8>(cfg, X, n, per, klo, khi, log_np1, hstat, gate)
              : d == 2 ? mcl_launch<2, 8>(cfg, X, n, per, klo, khi, log_np1, hstat, gate)
                       : mcl_launch<3, 8>(cfg, X, n, per, klo, khi, log_np1, hstat, gate);
        }
        FCB_CUDA(e);
        FCB_LAUNCHED("median_cluster_kernel");
        return FCB_OK;
    }
    return FCB_ENOTSUP;
}

extern "C" FCB_API int fcb_debug_mcl_timeline(unsigned long long* out) {
#ifdef MCL_TL
    cudaDeviceSynchronize();
    return cudaMemcpyFromSymbol(out, g_mcl_tl, sizeof(g_mcl_tl)) == cudaSuccess ? 128 : -1;
#else
    (void)out;
    return -1;
#endif
}

size_t median_ws_bytes(int n) {
    (void)n;
    return align_up(sizeof(MedState), 256);
}

int median_bandwidth(const double* X, int n, int d, double log_np1, double* hstat, const int* gate,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
    if (n < 1) return fail(FCB_EINPUT, "need at least one point");
    if (ws_bytes < median_ws_bytes(n)) return fail(FCB_EWORKSPACE, "median workspace too small");
    if (n == 1) {  // stein.py:73-74
        fixed_bandwidth_kernel<<<1, 32, 0, st>>>(1.0, hstat, gate);
        FCB_LAUNCHED("fixed_bandwidth_kernel");
        return FCB_OK;
    }
    MedState* ms = static_cast<MedState*>(ws);
    const unsigned long long N = (unsigned long long)n * (unsigned long long)n;
    const int nb = (n + MED_TILE - 1) / MED_TILE;
    const long long ntiles = (long long)nb * (nb + 1) / 2;
    if (median_cluster_launch(X, n, d, log_np1, hstat, gate, st) == FCB_OK) return FCB_OK;
    if (ntiles <= MED_COOP_TILES) {
        int per_sm = 0;
        const void* kern = d == 1 ? (const void*)median_coop_kernel<1>
                         : d == 2 ? (const void*)median_coop_kernel<2>
                                  : (const void*)median_coop_kernel<3>;
        FCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, MED_BLOCK, 0));
        if (per_sm >= 1 && d >= 1 && d <= 3) {
            int grid = (int)std::min<long long>(ntiles, (long long)per_sm * sm_count());
            unsigned long long klo = (N - 1ull) / 2ull, khi = N / 2ull;
            FCB_CUDA(cudaMemsetAsync(&ms->bar, 0, sizeof(GridBarrier), st));
            void* args[] = {(void*)&X, (void*)&n, (void*)&ms, (void*)&ntiles, (void*)&klo,
                            (void*)&khi, (void*)&log_np1, (void*)&hstat, (void*)&gate};
            FCB_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(MED_BLOCK), args, 0, st));
            FCB_LAUNCHED("median_coop_kernel");
            return FCB_OK;
        }
    }
    median_init_kernel<<<1, 256, 0, st>>>(ms, (N - 1ull) / 2ull, N / 2ull, gate);
    FCB_LAUNCHED("median_init_kernel");
    const int grid = (int)std::min<long long>(ntiles, 4LL * sm_count());
    for (int pass = 0; pass < MED_PASSES; ++pass) {
        switch (d) {
            case 1: median_hist_kernel<1><<<grid, MED_BLOCK, 0, st>>>(X, n, ms, pass, gate, 0, ntiles, 1); break;
            case 2: median_hist_kernel<2><<<grid, MED_BLOCK, 0, st>>>(X, n, ms, pass, gate, 0, ntiles, 1); break;
            case 3: median_hist_kernel<3><<<grid, MED_BLOCK, 0, st>>>(X, n, ms, pass, gate, 0, ntiles, 1); break;
            default: return fail(FCB_ENOTSUP, "dimension must be 1, 2 or 3");
        }
        FCB_LAUNCHED("median_hist_kernel");
    }
    median_finish_kernel<<<1, 32, 0, st>>>(ms, n, log_np1, hstat, gate);
    FCB_LAUNCHED("median_finish_kernel");
    return FCB_OK;
}

// ---- the M-sharded median (distributed.py): per radix pass, every rank
// histograms its share of the pair tiles, the caller all-reduces the
// histogram (MedState.hist, 2 x MED_BINS unsigned long long at byte offset
// median_hist_offset()), then every rank selects the same digit.
__global__ void median_select_kernel(MedState* st, int n, int pass, const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    median_select_block(st, n, pass);
}

long long median_tiles(int n) {
    const long long nb = (n + MED_TILE - 1) / MED_TILE;
    return nb * (nb + 1) / 2;
}

size_t median_hist_offset() { return offsetof(MedState, hist); }

int median_shard_init(int n, void* ws, size_t ws_bytes, const int* gate, cudaStream_t st) {
    if (n < 2) return fail(FCB_EINPUT, "sharded median needs n >= 2");
    if (ws_bytes < median_ws_bytes(n)) return fail(FCB_EWORKSPACE, "median workspace too small");
    const unsigned long long N = (unsigned long long)n * (unsigned long long)n;
    median_init_kernel<<<1, 256, 0, st>>>(static_cast<MedState*>(ws), (N - 1ull) / 2ull, N / 2ull,
                                          gate);
    FCB_LAUNCHED("median_init_kernel");
    return FCB_OK;
}

int median_shard_pass(const double* X, int n, int d, int pass, long long t_lo, long long t_hi,
                      void* ws, const int* gate, cudaStream_t st) {
    if (pass < 0 || pass >= MED_PASSES) return fail(FCB_EINPUT, "median pass out of range");
    MedState* ms = static_cast<MedState*>(ws);
    if (t_hi <= t_lo) return FCB_OK;
    const int grid = (int)std::min<long long>(t_hi - t_lo, 4LL * sm_count());
    switch (d) {
        case 1: median_hist_kernel<1><<<grid, MED_BLOCK, 0, st>>>(X, n, ms, pass, gate, t_lo, t_hi, 0); break;
        case 2: median_hist_kernel<2><<<grid, MED_BLOCK, 0, st>>>(X, n, ms, pass, gate, t_lo, t_hi, 0); break;
        case 3: median_hist_kernel<3><<<grid, MED_BLOCK, 0, st>>>(X, n, ms, pass, gate, t_lo, t_hi, 0); break;
        default: return fail(FCB_ENOTSUP, "dimension must be 1, 2 or 3");
    }
    FCB_LAUNCHED("median_hist_kernel");
    return FCB_OK;
}

int median_shard_select(int n, int pass, void* ws, const int* gate, cudaStream_t st) {
    median_select_kernel<<<1, MED_BLOCK, 0, st>>>(static_cast<MedState*>(ws), n, pass, gate);
    FCB_LAUNCHED("median_select_kernel");
    return FCB_OK;
}

int median_shard_finish(int n, double log_np1, double* hstat, void* ws, const int* gate,
                        cudaStream_t st) {
    median_finish_kernel<<<1, 32, 0, st>>>(static_cast<MedState*>(ws), n, log_np1, hstat, gate);
    FCB_LAUNCHED("median_finish_kernel");
    return FCB_OK;
}

// ---------------------------------------------------------------------------
// Stein flow
// ---------------------------------------------------------------------------
constexpr int SV_BLOCK = 256;
constexpr int SV_TILE = 256;
constexpr int SV_SUB = 8;
constexpr int SV_MAXCH = 64;
#ifndef FCB_SV_SCALAR
#define FCB_SV_SCALAR 0  // 1: fp32 SVGD sweeps use the scalar loop
#endif

template <typename Real>
struct alignas(sizeof(Real) * 4) SvCol {
    Real x[4];  // scaled centred coordinates (x[3] unused)
    Real w[4];  // w_j = s_j - (2/h) x'_j           (w[3] unused)
};

struct SvPlan {
    int n, nrb, nchunks, chunk_len, items, n8;
};

// rows n (queries), columns nc (sources; default: the same n points)
static SvPlan sv_plan(int n, int rpt, int grid, int nc = -1) {
    SvPlan p{};
    p.n = n;
    if (nc < 0) nc = n;
    p.n8 = (nc + SV_SUB - 1) / SV_SUB * SV_SUB;
    const int br = SV_BLOCK * rpt;
    p.nrb = (n + br - 1) / br;
    const int maxch = std::max(1, std::min(SV_MAXCH, p.n8 / 64));
    int best = 1;
    double best_eff = -1.0;
    for (int k = 1; k <= maxch; ++k) {
        const long items = (long)p.nrb * k;
        const long waves = (items + grid - 1) / grid;
        const double eff = (double)items / (double)(waves * grid);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = k;
        }
        if (eff > 0.97) break;
    }
    int cl = (p.n8 + best - 1) / best;
    cl = (cl + SV_SUB - 1) / SV_SUB * SV_SUB;
    p.chunk_len = cl;
    p.nchunks = (p.n8 + cl - 1) / cl;
    p.items = p.nrb * p.nchunks;
    return p;
}

template <typename Real, int D>
__global__ void sv_pack_kernel(const double* __restrict__ X, int n, int n8,
                               const double* __restrict__ score, const double* __restrict__ hstat,
                               const double* __restrict__ centre, SvCol<Real>* __restrict__ cols,
                               Vec4<Real>* __restrict__ rows, const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    const double h = hstat[0];
    const double unit = (sizeof(Real) == 4) ? kLog2e : 1.0;
    const double sc = sqrt(unit / h);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n8; j += gridDim.x * blockDim.x) {
        SvCol<Real> c{};
        Vec4<Real> r{};
        if (j < n) {
            Real xs[3] = {0, 0, 0};
            for (int q = 0; q < D; ++q) {
                const double xc = X[(size_t)j * D + q] - centre[q];
                c.x[q] = (Real)(xc * sc);
                c.w[q] = (Real)(score[(size_t)j * D + q] - (2.0 / h) * xc);
                xs[q] = c.x[q];
            }
            r = Vec4<Real>{xs[0], xs[1], xs[2], 0};
            rows[j] = r;
        } else {
            for (int q = 0; q < 4; ++q) {
                c.x[q] = (Real)1e30;  // padding: distance -> inf, kernel weight -> 0
                c.w[q] = 0;
            }
        }
        cols[j] = c;
    }
}

template <typename Real, int D, int RPT>
__global__ void __launch_bounds__(SV_BLOCK) sv_sweep_kernel(SvPlan pl,
                                                            const Vec4<Real>* __restrict__ rows,
                                                            const SvCol<Real>* __restrict__ cols,
                                                            Real* __restrict__ part,
                                                            const int* gate) {
    using U = Units<Real>;
    __shared__ SvCol<Real> tile[SV_TILE];
    if (gate && *((volatile const int*)gate) != 0) return;
    const int n = pl.n;
    for (int item = blockIdx.x; item < pl.items; item += gridDim.x) {
        const int rb = item % pl.nrb, ch = item / pl.nrb;
        const int c0 = ch * pl.chunk_len, c1 = min(c0 + pl.chunk_len, pl.n8);
        const int row0 = rb * SV_BLOCK * RPT;
        Real x[RPT][D], ks[RPT], acc[RPT][D];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int i = min(row0 + r * SV_BLOCK + threadIdx.x, n - 1);
            const Vec4<Real> v = rows[i];
#pragma unroll
            for (int q = 0; q < D; ++q) {
                x[r][q] = vget(v, q);
                acc[r][q] = 0;
            }
            ks[r] = 0;
        }
        for (int t0 = c0; t0 < c1; t0 += SV_TILE) {
            const int len = min(SV_TILE, c1 - t0);
            __syncthreads();
            for (int k = threadIdx.x; k < len; k += SV_BLOCK) tile[k] = cols[t0 + k];
            __syncthreads();
            for (int c = 0; c < len; c += SV_SUB) {
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    Real ts = 0, ta[D];
#pragma unroll
                    for (int q = 0; q < D; ++q) ta[q] = 0;
#pragma unroll
                    for (int k = 0; k < SV_SUB; ++k) {
                        const SvCol<Real>& cc = tile[c + k];
                        Real d2 = 0;
#pragma unroll
                        for (int q = 0; q < D; ++q) {
                            const Real df = x[r][q] - cc.x[q];
                            d2 = fma(df, df, d2);
                        }
                        const Real e = U::expu(-d2);
                        ts += e;
#pragma unroll
                        for (int q = 0; q < D; ++q) ta[q] = fma(e, cc.w[q], ta[q]);
                    }
                    ks[r] += ts;
#pragma unroll
                    for (int q = 0; q < D; ++q) acc[r][q] += ta[q];
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int i = row0 + r * SV_BLOCK + threadIdx.x;
            if (i < n) {
                part[((size_t)ch * (D + 1)) * n + i] = ks[r];
#pragma unroll
                for (int q = 0; q < D; ++q) part[((size_t)ch * (D + 1) + 1 + q) * n + i] = acc[r][q];
            }
        }
    }
}

// fp32 sweep with packed FADD2/FFMA2: columns staged structure-of-arrays
// (-x~_j and w_j per coordinate, float4 quads), two columns per packed op, the
// direct form k = 2^-(|x~_i - x~_j|^2) with the negation folded into the
// MUFU.EX2 operand.  ~6 issue slots per pair (scalar loop: ~11).
template <int D, int RPT>
__global__ void __launch_bounds__(SV_BLOCK) sv_sweep_f32_kernel(SvPlan pl,
                                                                const Vec4<float>* __restrict__ rows,
                                                                const SvCol<float>* __restrict__ cols,
                                                                float* __restrict__ part,
                                                                const int* gate) {
    __shared__ __align__(16) float s_y[D][SV_TILE];
    __shared__ __align__(16) float s_w[D][SV_TILE];
    if (gate && *((volatile const int*)gate) != 0) return;
    const int n = pl.n;
    for (int item = blockIdx.x; item < pl.items; item += gridDim.x) {
        const int rb = item % pl.nrb, ch = item / pl.nrb;
        const int c0 = ch * pl.chunk_len, c1 = min(c0 + pl.chunk_len, pl.n8);
        const int row0 = rb * SV_BLOCK * RPT;
        float2 x2[RPT][D], ks2[RPT], acc2[RPT][D];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int i = min(row0 + r * SV_BLOCK + threadIdx.x, n - 1);
            const Vec4<float> v = rows[i];
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const float xv = vget(v, q);
                x2[r][q] = make_float2(xv, xv);
                acc2[r][q] = make_float2(0.f, 0.f);
            }
            ks2[r] = make_float2(0.f, 0.f);
        }
        for (int t0 = c0; t0 < c1; t0 += SV_TILE) {
            const int len = min(SV_TILE, c1 - t0);
            __syncthreads();
            for (int k = threadIdx.x; k < len; k += SV_BLOCK) {
                const SvCol<float> c = cols[t0 + k];
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    s_y[q][k] = -c.x[q];
                    s_w[q][k] = c.w[q];
                }
            }
            __syncthreads();
            for (int c = 0; c < len; c += SV_SUB) {
                float y[D][8], w[D][8];
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    const float4 a = *reinterpret_cast<const float4*>(&s_y[q][c]);
                    const float4 b = *reinterpret_cast<const float4*>(&s_y[q][c + 4]);
                    y[q][0] = a.x; y[q][1] = a.y; y[q][2] = a.z; y[q][3] = a.w;
                    y[q][4] = b.x; y[q][5] = b.y; y[q][6] = b.z; y[q][7] = b.w;
                    const float4 e = *reinterpret_cast<const float4*>(&s_w[q][c]);
                    const float4 f = *reinterpret_cast<const float4*>(&s_w[q][c + 4]);
                    w[q][0] = e.x; w[q][1] = e.y; w[q][2] = e.z; w[q][3] = e.w;
                    w[q][4] = f.x; w[q][5] = f.y; w[q][6] = f.z; w[q][7] = f.w;
                }
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    float2 e[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float2 d2 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int q = 0; q < D; ++q) {
                            const float2 df = __fadd2_rn(x2[r][q], make_float2(y[q][2 * u], y[q][2 * u + 1]));
                            d2 = __ffma2_rn(df, df, d2);
                        }
                        e[u] = make_float2(ex2_approx(-d2.x), ex2_approx(-d2.y));
                    }
                    ks2[r] = __fadd2_rn(ks2[r], __fadd2_rn(__fadd2_rn(e[0], e[1]), __fadd2_rn(e[2], e[3])));
#pragma unroll
                    for (int q = 0; q < D; ++q)
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            acc2[r][q] = __ffma2_rn(e[u], make_float2(w[q][2 * u], w[q][2 * u + 1]),
                                                    acc2[r][q]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int i = row0 + r * SV_BLOCK + threadIdx.x;
            if (i < n) {
                part[((size_t)ch * (D + 1)) * n + i] = ks2[r].x + ks2[r].y;
#pragma unroll
                for (int q = 0; q < D; ++q)
                    part[((size_t)ch * (D + 1) + 1 + q) * n + i] = acc2[r][q].x + acc2[r][q].y;
            }
        }
    }
}

// Launch the sweep of the precision (fp32: the packed kernel).
template <typename Real, int D, int RPT>
static void sv_sweep_launch(const SvPlan& pl, int grid, const void* rows, const void* cols,
                            void* part, const int* gate, cudaStream_t st) {
    if constexpr (sizeof(Real) == 4 && !FCB_SV_SCALAR) {
        sv_sweep_f32_kernel<D, RPT><<<grid, SV_BLOCK, 0, st>>>(
            pl, static_cast<const Vec4<float>*>(rows), static_cast<const SvCol<float>*>(cols),
            static_cast<float*>(part), gate);
    } else {
        sv_sweep_kernel<Real, D, RPT><<<grid, SV_BLOCK, 0, st>>>(
            pl, static_cast<const Vec4<Real>*>(rows), static_cast<const SvCol<Real>*>(cols),
            static_cast<Real*>(part), gate);
    }
}

template <typename Real, int D>
__global__ void sv_merge_kernel(SvPlan pl, const Real* __restrict__ part,
                                const double* __restrict__ X, const double* __restrict__ hstat,
                                const double* __restrict__ centre, double* __restrict__ out,
                                const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    const int n = pl.n;
    const double h = hstat[0];
    const double two_over_h = 2.0 / h, inv_n = 1.0 / n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double K = 0.0, A[D];
#pragma unroll
        for (int q = 0; q < D; ++q) A[q] = 0.0;
        for (int ch = 0; ch < pl.nchunks; ++ch) {
            K += (double)part[((size_t)ch * (D + 1)) * n + i];
#pragma unroll
            for (int q = 0; q < D; ++q) A[q] += (double)part[((size_t)ch * (D + 1) + 1 + q) * n + i];
        }
#pragma unroll
        for (int q = 0; q < D; ++q) {
            const double xc = X[(size_t)i * D + q] - centre[q];
            out[(size_t)i * D + q] = inv_n * (A[q] + two_over_h * xc * K);
        }
    }
}

constexpr int SV_RPT_F32 = 4;  // packed loop: 4 rows per thread halve the shared-memory loads per pair
constexpr int SV_RPT_F64 = 1;

// Sharded sources (fcb_stein_partial): query rows are all n points, source
// columns the points [col0, col0 + nc); centred on X[0] like stein_run.
template <typename Real, int D>
__global__ void sv_pack_range_kernel(const double* __restrict__ X, int n, int col0, int nc,
                                     int nc8, const double* __restrict__ score,
                                     const double* __restrict__ hstat,
                                     SvCol<Real>* __restrict__ cols, Vec4<Real>* __restrict__ rows,
                                     const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    const double h = hstat[0];
    const double unit = (sizeof(Real) == 4) ? kLog2e : 1.0;
    const double sc = sqrt(unit / h);
    const int tot = max(n, nc8);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < tot; j += gridDim.x * blockDim.x) {
        if (j < n) {
            Real xs[3] = {0, 0, 0};
            for (int q = 0; q < D; ++q) xs[q] = (Real)((X[(size_t)j * D + q] - X[q]) * sc);
            rows[j] = Vec4<Real>{xs[0], xs[1], xs[2], 0};
        }
        if (j < nc8) {
            SvCol<Real> c{};
            if (j < nc) {
                const size_t g = (size_t)(col0 + j);
                for (int q = 0; q < D; ++q) {
                    const double xc = X[g * D + q] - X[q];
                    c.x[q] = (Real)(xc * sc);
                    c.w[q] = (Real)(score[g * D + q] - (2.0 / h) * xc);
                }
            } else {
                for (int q = 0; q < 4; ++q) {
                    c.x[q] = (Real)1e30;
                    c.w[q] = 0;
                }
            }
            cols[j] = c;
        }
    }
}

// Raw per-row sums over the source chunks: out[i] = {sum_j k_ij, sum_j k_ij w_j}.
template <typename Real, int D>
__global__ void sv_merge_raw_kernel(SvPlan pl, const Real* __restrict__ part,
                                    double* __restrict__ out, const int* gate) {
    if (gate && *((volatile const int*)gate) != 0) return;
    const int n = pl.n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double K = 0.0, A[D];
#pragma unroll
        for (int q = 0; q < D; ++q) A[q] = 0.0;
        for (int ch = 0; ch < pl.nchunks; ++ch) {
            K += (double)part[((size_t)ch * (D + 1)) * n + i];
#pragma unroll
            for (int q = 0; q < D; ++q) A[q] += (double)part[((size_t)ch * (D + 1) + 1 + q) * n + i];
        }
        out[(size_t)i * (D + 1)] = K;
#pragma unroll
        for (int q = 0; q < D; ++q) out[(size_t)i * (D + 1) + 1 + q] = A[q];
    }
}

struct SvWs {
    double* centre;
    void* cols;
    void* rows;
    void* part;
    size_t total;
};

static SvWs sv_layout(int precision, int n, int d, SvPlan pl, void* ws, size_t bytes) {
    Arena ar(ws, bytes);
    SvWs L{};
    L.centre = ar.take<double>(4);
    if (precision == FCB_FP64) {
        L.cols = ar.take<SvCol<double>>(pl.n8);
        L.rows = ar.take<Vec4<double>>(n);
        L.part = ar.take<double>((size_t)pl.nchunks * (d + 1) * n);
    } else {
        L.cols = ar.take<SvCol<float>>(pl.n8);
        L.rows = ar.take<Vec4<float>>(n);
        L.part = ar.take<float>((size_t)pl.nchunks * (d + 1) * n);
    }
    L.total = ar.off + 256;
    return L;
}

static int sv_grid() { return 2 * sm_count(); }

size_t stein_ws_bytes(int precision, int n, int d) {
    const int rpt = precision == FCB_FP64 ? SV_RPT_F64 : SV_RPT_F32;
    SvPlan pl = sv_plan(n, rpt, sv_grid());
    return sv_layout(precision, n, d, pl, nullptr, 0).total;
}

template <typename Real, int D, int RPT>
static int stein_run(const double* X, int n, const double* scores, const double* hstat,
                     double* out, const int* gate, void* ws, size_t ws_bytes, cudaStream_t st) {
    const int precision = sizeof(Real) == 8 ? FCB_FP64 : FCB_FP32;
    SvPlan pl = sv_plan(n, RPT, sv_grid());
    SvWs L = sv_layout(precision, n, D, pl, ws, ws_bytes);
    if (L.total > ws_bytes) return fail(FCB_EWORKSPACE, "stein workspace too small");
    // centre on the first point: exactly coincident clouds (the degenerate
    // median case of stein.py:101-103) then have x' == 0 bit-exactly
    const double* centre = X;
    const int pb = std::max(1, std::min(4 * sm_count(), (pl.n8 + 255) / 256));
    sv_pack_kernel<Real, D><<<pb, 256, 0, st>>>(X, n, pl.n8, scores, hstat, centre,
                                               static_cast<SvCol<Real>*>(L.cols),
                                               static_cast<Vec4<Real>*>(L.rows), gate);
    FCB_LAUNCHED("sv_pack_kernel");
    const int grid = std::min(pl.items, sv_grid());
    sv_sweep_launch<Real, D, RPT>(pl, grid, L.rows, L.cols, L.part, gate, st);
    FCB_LAUNCHED("sv_sweep_kernel");
    const int mb = std::max(1, std::min(4 * sm_count(), (n + 255) / 256));
    sv_merge_kernel<Real, D><<<mb, 256, 0, st>>>(pl, static_cast<const Real*>(L.part), X, hstat,
                                                centre, out, gate);
    FCB_LAUNCHED("sv_merge_kernel");
    return FCB_OK;
}

int stein_flow(int precision, const double* X, int n, int d, const double* scores,
               const double* hstat, double* out, const int* gate, void* ws, size_t ws_bytes,
               cudaStream_t st) {
    if (n < 1) return fail(FCB_EINPUT, "need at least one point");
#define FCB_SV_CASE(DD)                                                                          \
    if (d == DD) {                                                                               \
        if (precision == FCB_FP64)                                                               \
            return stein_run<double, DD, SV_RPT_F64>(X, n, scores, hstat, out, gate, ws,         \
                                                     ws_bytes, st);                              \
        return stein_run<float, DD, SV_RPT_F32>(X, n, scores, hstat, out, gate, ws, ws_bytes,   \
                                                st);                                             \
    }
    FCB_SV_CASE(1)
    FCB_SV_CASE(2)
    FCB_SV_CASE(3)
#undef FCB_SV_CASE
    return fail(FCB_ENOTSUP, "dimension must be 1, 2 or 3");
}

size_t stein_partial_ws_bytes(int precision, int n, int nc, int d) {
    const int rpt = precision == FCB_FP64 ? SV_RPT_F64 : SV_RPT_F32;
    SvPlan pl = sv_plan(n, rpt, sv_grid(), nc);
    return sv_layout(precision, std::max(n, pl.n8), d, pl, nullptr, 0).total;
}

template <typename Real, int D, int RPT>
static int stein_partial_run(const double* X, int n, int col0, int nc, const double* scores,
                             const double* hstat, double* out, const int* gate, void* ws,
                             size_t ws_bytes, cudaStream_t st) {
    const int precision = sizeof(Real) == 8 ? FCB_FP64 : FCB_FP32;
    SvPlan pl = sv_plan(n, RPT, sv_grid(), nc);
    SvWs L = sv_layout(precision, std::max(n, pl.n8), D, pl, ws, ws_bytes);
    if (L.total > ws_bytes) return fail(FCB_EWORKSPACE, "stein_partial workspace too small");
    const int pb = std::max(1, std::min(4 * sm_count(), (std::max(n, pl.n8) + 255) / 256));
    sv_pack_range_kernel<Real, D><<<pb, 256, 0, st>>>(X, n, col0, nc, pl.n8, scores, hstat,
                                                     static_cast<SvCol<Real>*>(L.cols),
                                                     static_cast<Vec4<Real>*>(L.rows), gate);
    FCB_LAUNCHED("sv_pack_range_kernel");
    const int grid = std::min(pl.items, sv_grid());
    sv_sweep_launch<Real, D, RPT>(pl, grid, L.rows, L.cols, L.part, gate, st);
    FCB_LAUNCHED("sv_sweep_kernel");
    const int mb = std::max(1, std::min(4 * sm_count(), (n + 255) / 256));
    sv_merge_raw_kernel<Real, D><<<mb, 256, 0, st>>>(pl, static_cast<const Real*>(L.part), out,
                                                    gate);
    FCB_LAUNCHED("sv_merge_raw_kernel");
    return FCB_OK;
}

int stein_partial(int precision, const double* X, int n, int d, int col0, int nc,
                  const double* scores, const double* hstat, double* out, const int* gate,
                  void* ws, size_t ws_bytes, cudaStream_t st) {
    if (n < 1 || nc < 1 || col0 < 0 || col0 + nc > n)
        return fail(FCB_EINPUT, "stein_partial: bad source range");
#define FCB_SP_CASE(DD)                                                                         \
    if (d == DD) {                                                                              \
        if (precision == FCB_FP64)                                                              \
            return stein_partial_run<double, DD, SV_RPT_F64>(X, n, col0, nc, scores, hstat,     \
                                                             out, gate, ws, ws_bytes, st);      \
        return stein_partial_run<float, DD, SV_RPT_F32>(X, n, col0, nc, scores, hstat, out,     \
                                                        gate, ws, ws_bytes, st);                \
    }
    FCB_SP_CASE(1)
    FCB_SP_CASE(2)
    FCB_SP_CASE(3)
#undef FCB_SP_CASE
    return fail(FCB_ENOTSUP, "dimension must be 1, 2 or 3");
}

// ---------------------------------------------------------------------------
// planner composite: bandwidth, score, flow, convergence hook
// ---------------------------------------------------------------------------
constexpr int SFIN_BLOCK = 1024;
__global__ void __launch_bounds__(SFIN_BLOCK)
    stein_finalize_kernel(const double* __restrict__ flow, int n, int d,
                          const double* __restrict__ hstat, double* fstat, int* plan_state,
                          int iteration, double* flow_log, double conv_tol) {
    __shared__ double scratch[32];
    if (plan_state && *((volatile int*)plan_state) != 0) return;
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += SFIN_BLOCK) {
        double sq = 0.0;
        for (int q = 0; q < d; ++q) {
            const double v = flow[(size_t)i * d + q];
            sq += v * v;
        }
        acc += sqrt(sq);
    }
    const double total = block_sum<SFIN_BLOCK>(acc, scratch);
    if (threadIdx.x == 0) {
        const double mean_mag = total / n;
        fstat[0] = 0.0;
        fstat[1] = 1.0;
        fstat[2] = 0.0;
        fstat[3] = mean_mag;
        fstat[4] = hstat[0];
        fstat[5] = hstat[2];
        fstat[6] = hstat[1];
        fstat[7] = 0.0;
        if (plan_state) {
            double* lg = flow_log + 4 * (size_t)iteration;
            lg[0] = mean_mag;
            lg[1] = hstat[0];
            lg[2] = hstat[2];
            lg[3] = hstat[1];
            plan_state[FCB_STATE_FLOWS] = iteration + 1;
            if (mean_mag < conv_tol) plan_state[FCB_STATE_STOP] = 1;
        }
    }
}

struct SfWs {
    double* hstat;
    double* scores;
    void* med;
    void* sv;
    size_t sv_bytes, total;
};

static SfWs sf_layout(int precision, int n, int d, void* ws, size_t bytes) {
    Arena ar(ws, bytes);
    SfWs L{};
    L.hstat = ar.take<double>(4);
    L.scores = ar.take<double>((size_t)n * d);
    L.med = ar.take<char>(median_ws_bytes(n));
    L.sv_bytes = stein_ws_bytes(precision, n, d);
    L.sv = ar.take<char>(L.sv_bytes);
    L.total = ar.off + 256;
    return L;
}

size_t stein_flow_full_ws_bytes(int precision, int n, int d) {
    return sf_layout(precision, n, d, nullptr, 0).total;
}

int stein_flow_full(int precision, const double* X, int n, int d, int k, const double* prm,
                    double bandwidth_fixed, double log_np1, double* flow, double* fstat,
                    int* plan_state, int iteration, double* flow_log, double conv_tol, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
    SfWs L = sf_layout(precision, n, d, ws, ws_bytes);
    if (L.total > ws_bytes) return fail(FCB_EWORKSPACE, "stein_flow_full workspace too small");
    int rc;
    if (bandwidth_fixed > 0.0) {
        fixed_bandwidth_kernel<<<1, 32, 0, st>>>(bandwidth_fixed, L.hstat, plan_state);
        FCB_LAUNCHED("fixed_bandwidth_kernel");
    } else {
        rc = median_bandwidth(X, n, d, log_np1, L.hstat, plan_state, L.med, median_ws_bytes(n), st);
        if (rc) return rc;
    }
    rc = gmm_eval(X, n, d, k, prm, L.scores, nullptr, plan_state, st);
    if (rc) return rc;
    rc = stein_flow(precision, X, n, d, L.scores, L.hstat, flow, plan_state, L.sv, L.sv_bytes, st);
    if (rc) return rc;
    stein_finalize_kernel<<<1, SFIN_BLOCK, 0, st>>>(flow, n, d, L.hstat, fstat, plan_state,
                                                    iteration, flow_log, conv_tol);
    FCB_LAUNCHED("stein_finalize_kernel");
    return FCB_OK;
}

}  // namespace fcb
