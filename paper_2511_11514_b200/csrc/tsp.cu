// tsp.cu -- the TSP-waypoint baseline's tour construction on the GPU
// (reference tsp.py:76-147: nearest-neighbour order from a seeded start, then
// first-improving 2-opt moves until none improves or the budget runs out).
//
// One CTA per problem (BASELINE config 5 plans 4096 independent problems):
// the points, the current path P = points[order] and the path's edge lengths
// live in shared memory.
//   nearest neighbour  n-1 steps; each a block-wide argmin over the remaining
//                      points of |p - p_cur|^2 (ties -> lowest index, as
//                      np.argmin), two shared-memory atomicMin rounds.
//   2-opt              the lexicographically first (i, j) with
//                      delta = (|P_j - P_{i-1}| - |P_i - P_{i-1}|)
//                            + (|P_{j+1} - P_i| - |P_{j+1} - P_j|) < -1e-12
//                      (missing end edges count zero): R rows of candidates
//                      are evaluated per block step and the first hit wins by
//                      an atomicMin on the key i*n + j; the move reverses
//                      P[i..j] in place and refreshes the edge lengths there.
// The arithmetic is the reference's, operation for operation, in IEEE double
// with no contraction (__dadd_rn / __dmul_rn / sqrt), so the move sequence and
// the final order are identical to the reference's.
#include <algorithm>

#include "fcb_internal.cuh"

namespace fcb {

constexpr int TSP_BLOCK = 1024;
constexpr double TSP_EPS = 1e-12;  // tsp.py:27 IMPROVEMENT_EPS

template <int D>
__device__ __forceinline__ double tsp_sq(const double* a, const double* b) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
        const double df = __dsub_rn(a[q], b[q]);
        const double sq = __dmul_rn(df, df);
        s = (q == 0) ? sq : __dadd_rn(s, sq);
    }
    return s;
}

template <int D>
__device__ __forceinline__ double tsp_dist(const double* a, const double* b) {
    return __dsqrt_rn(tsp_sq<D>(a, b));
}

template <int D>
__global__ void __launch_bounds__(TSP_BLOCK)
    tsp_tour_kernel(const double* __restrict__ pts_all, int n, const int* __restrict__ starts,
                    int budget, int rows_per_step, int* __restrict__ order_all,
                    int* __restrict__ moves_out) {
    extern __shared__ __align__(16) double tsp_smem[];
    double* pts = tsp_smem;                  // n * D, original point order
    double* P = pts + (size_t)n * D;         // n * D, current path
    double* edge = P + (size_t)n * D;        // n: |P[k+1] - P[k]| (last: 0)
    int* ord = reinterpret_cast<int*>(edge + n);
    int* rem = ord + n;
    __shared__ unsigned long long s_key;
    __shared__ int s_idx;
    const int tid = threadIdx.x;
    const int b = blockIdx.x;
    const double* src = pts_all + (size_t)b * n * D;
    for (int e = tid; e < n * D; e += TSP_BLOCK) pts[e] = src[e];
    for (int j = tid; j < n; j += TSP_BLOCK) rem[j] = 1;
    __syncthreads();

    // ---- nearest-neighbour order (tsp.py:76-89) ---------------------------------
    int cur = starts[b];
    if (tid == 0) {
        ord[0] = cur;
        rem[cur] = 0;
    }
    __syncthreads();
    for (int k = 1; k < n; ++k) {
        if (tid == 0) {
            s_key = ~0ull;
            s_idx = 0x7fffffff;
        }
        __syncthreads();
        const double* pc = pts + (size_t)cur * D;
        for (int j = tid; j < n; j += TSP_BLOCK)
            if (rem[j])
                atomicMin(&s_key, (unsigned long long)__double_as_longlong(tsp_sq<D>(pts + (size_t)j * D, pc)));
        __syncthreads();
        const unsigned long long best = s_key;
        for (int j = tid; j < n; j += TSP_BLOCK)
            if (rem[j] &&
                (unsigned long long)__double_as_longlong(tsp_sq<D>(pts + (size_t)j * D, pc)) == best)
                atomicMin(&s_idx, j);
        __syncthreads();
        cur = s_idx;
        if (tid == 0) {
            ord[k] = cur;
            rem[cur] = 0;
        }
        __syncthreads();
    }

    // ---- path and edges ----------------------------------------------------------
    for (int e = tid; e < n * D; e += TSP_BLOCK) P[e] = pts[(size_t)ord[e / D] * D + e % D];
    __syncthreads();
    for (int k = tid; k < n; k += TSP_BLOCK)
        edge[k] = (k + 1 < n) ? tsp_dist<D>(P + (size_t)(k + 1) * D, P + (size_t)k * D) : 0.0;
    __syncthreads();

    // ---- first-improving 2-opt (tsp.py:92-117, 140-146) ---------------------------
    int moves = 0;
    while (moves < budget) {
        int found_i = -1, found_j = -1;
        for (int i0 = 0; i0 < n - 1; i0 += rows_per_step) {
            if (tid == 0) s_key = ~0ull;
            __syncthreads();
            const int i1 = min(i0 + rows_per_step, n - 1);
            for (int i = i0; i < i1; ++i) {
                const double* Pi = P + (size_t)i * D;
                const double left_old = (i > 0) ? tsp_dist<D>(Pi, Pi - D) : 0.0;
                for (int j = i + 1 + tid; j < n; j += TSP_BLOCK) {
                    const double* Pj = P + (size_t)j * D;
                    const double left_new = (i > 0) ? tsp_dist<D>(Pj, Pi - D) : 0.0;
                    const double right_new = (j + 1 < n) ? tsp_dist<D>(Pj + D, Pi) : 0.0;
                    const double right_old = edge[j];
                    const double delta = __dadd_rn(__dsub_rn(left_new, left_old),
                                                   __dsub_rn(right_new, right_old));
                    if (delta < -TSP_EPS)
                        atomicMin(&s_key, (unsigned long long)i * (unsigned long long)n + j);
                }
            }
            __syncthreads();
            const unsigned long long key = s_key;
            if (key != ~0ull) {
                found_i = (int)(key / (unsigned long long)n);
                found_j = (int)(key % (unsigned long long)n);
                break;
            }
        }
        if (found_i < 0) break;
        // reverse P[i..j] (and the order) in place
        const int i = found_i, j = found_j, half = (j - i + 1) / 2;
        for (int s = tid; s < half; s += TSP_BLOCK) {
            const int a = i + s, c = j - s;
            const int t = ord[a];
            ord[a] = ord[c];
            ord[c] = t;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double v = P[(size_t)a * D + q];
                P[(size_t)a * D + q] = P[(size_t)c * D + q];
                P[(size_t)c * D + q] = v;
            }
        }
        __syncthreads();
        // edges k in [i-1, j] changed (reversed interior edges keep their length,
        // but recomputing them is cheaper than reasoning about it)
        for (int k = max(i - 1, 0) + tid; k <= j; k += TSP_BLOCK)
            edge[k] = (k + 1 < n) ? tsp_dist<D>(P + (size_t)(k + 1) * D, P + (size_t)k * D) : 0.0;
        __syncthreads();
        ++moves;
    }
    int* out = order_all + (size_t)b * n;
    for (int k = tid; k < n; k += TSP_BLOCK) out[k] = ord[k];
    if (tid == 0 && moves_out) moves_out[b] = moves;
}

static size_t tsp_smem_bytes(int n, int d) {
    return (size_t)n * (2 * d + 1) * sizeof(double) + 2 * (size_t)n * sizeof(int);
}

int tsp_tours(const double* pts, int batch, int n, int d, const int* starts, int budget,
              int* order, int* moves, cudaStream_t st) {
    if (batch < 1 || n < 2) return fail(FCB_EINPUT, "tsp: need at least two points per problem");
    if (d < 1 || d > 3) return fail(FCB_ENOTSUP, "tsp: dimension must be 1, 2 or 3");
    const size_t smem = tsp_smem_bytes(n, d);
    int lim = 0;
    FCB_CUDA(cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, current_device()));
    if (smem + 64 > (size_t)lim) return fail(FCB_ENOTSUP, "tsp: point set does not fit in shared memory");
    // rows per block step: about 4 candidates per thread
    const int rows = std::max(1, std::min(64, 4 * TSP_BLOCK / n));
    switch (d) {
#define FCB_TSP_CASE(DD)                                                                        \
    case DD: {                                                                                  \
        FCB_CUDA(cudaFuncSetAttribute(tsp_tour_kernel<DD>,                                     \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        tsp_tour_kernel<DD><<<batch, TSP_BLOCK, smem, st>>>(pts, n, starts, budget, rows, order, \
                                                            moves);                            \
        break;                                                                                  \
    }
        FCB_TSP_CASE(1)
        FCB_TSP_CASE(2)
        FCB_TSP_CASE(3)
#undef FCB_TSP_CASE
    }
    FCB_LAUNCHED("tsp_tour_kernel");
    return FCB_OK;
}

}  // namespace fcb

extern "C" FCB_API int fcb_tsp_tours(const double* points, int batch, int n, int d,
                                     const int* starts, int budget, int* order, int* moves,
                                     fcb_stream_t stream) {
    return fcb::tsp_tours(points, batch, n, d, starts, budget, order, moves,
                          static_cast<cudaStream_t>(stream));
}
