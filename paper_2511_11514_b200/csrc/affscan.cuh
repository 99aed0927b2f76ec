// affscan.cuh -- parallel scans of affine recurrences over time, one thread
// per time step.
//
//   forward : s_{k+1} = M_k s_k + c_k     (s_0 given)      k = 0..T-1
//   backward: e_k     = M_k e_{k+1} + c_k (e_T given)      k = T-1..0
//
// Three launches, no grid-wide synchronisation:
//   K1  every CTA owns AS_BLK consecutive steps; each thread builds its step
//       map (all per-step loads in flight at once), then a Hillis-Steele scan
//       in shared memory composes the block's maps; the block aggregate goes
//       to global memory.
//   K2  one CTA scans the block aggregates and writes the state entering each
//       block.
//   K3  every CTA repeats its in-block scan, applies it to its entry state and
//       hands each step's (state before, state after) to a consumer functor;
//       consumer return values are summed per block in a fixed order.
// Used by the planner for the linear-model rollout and both passes of the
// LQR affine phase (lqr_split.cuh).
#pragma once

#include "fcb_internal.cuh"

namespace fcb {

constexpr int AS_BLK = 128;

template <int N>
struct AMap {
    double M[N][N];
    double c[N];
};

template <int N>
__device__ __forceinline__ void amap_identity(AMap<N>& a) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        a.c[i] = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) a.M[i][j] = (i == j) ? 1.0 : 0.0;
    }
}

// out = later o earlier (apply `earlier` first)
template <int N>
__device__ __forceinline__ void amap_compose(const AMap<N>& later, const AMap<N>& earlier,
                                             AMap<N>& out) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double cc = later.c[i];
#pragma unroll
        for (int q = 0; q < N; ++q) cc += later.M[i][q] * earlier.c[q];
        out.c[i] = cc;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += later.M[i][q] * earlier.M[q][j];
            out.M[i][j] = s;
        }
    }
}

template <int N>
__device__ __forceinline__ void amap_apply(const AMap<N>& a, const double* x, double* y) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double s = a.c[i];
#pragma unroll
        for (int q = 0; q < N; ++q) s += a.M[i][q] * x[q];
        y[i] = s;
    }
}

template <int N>
__device__ __forceinline__ void amap_copy_to(double* __restrict__ dst, const AMap<N>& a) {
#pragma unroll
    for (int i = 0; i < N * N; ++i) dst[i] = (&a.M[0][0])[i];
#pragma unroll
    for (int i = 0; i < N; ++i) dst[N * N + i] = a.c[i];
}

template <int N>
__device__ __forceinline__ void amap_copy_from(const double* __restrict__ src, AMap<N>& a) {
#pragma unroll
    for (int i = 0; i < N * N; ++i) (&a.M[0][0])[i] = src[i];
#pragma unroll
    for (int i = 0; i < N; ++i) a.c[i] = src[N * N + i];
}

template <int N>
constexpr int amap_doubles() {
    return N * N + N;
}

// In-block inclusive scan (prefix for FWD, suffix for BWD) of the maps of
// steps blockIdx.x*AS_BLK + t; returns this thread's inclusive map.  buf:
// shared memory of 2*AS_BLK*amap_doubles<N>() doubles.
template <int N, bool FWD, class MapFn>
__device__ __forceinline__ void block_scan(const MapFn& mapf, int T, double* buf, AMap<N>& mine) {
    constexpr int AD = amap_doubles<N>();
    const int t = threadIdx.x;
    const int k = blockIdx.x * AS_BLK + t;
    if (k < T) mapf(k, mine);
    else amap_identity<N>(mine);
    double* cur = buf;
    double* nxt = buf + AS_BLK * AD;
    amap_copy_to<N>(cur + t * AD, mine);
    __syncthreads();
    for (int s = 1; s < AS_BLK; s <<= 1) {
        const int o = FWD ? t - s : t + s;
        if (o >= 0 && o < AS_BLK) {
            AMap<N> other, res;
            amap_copy_from<N>(cur + o * AD, other);
            // FWD: mine covers (t-s, t], other the earlier steps
            // BWD: mine covers [t, t+s), other the later steps (applied first)
            amap_compose<N>(mine, other, res);
            mine = res;
        }
        amap_copy_to<N>(nxt + t * AD, mine);
        __syncthreads();
        double* tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
}

template <int N, bool FWD, class MapFn>
__global__ void __launch_bounds__(AS_BLK) affscan_k1(int T, MapFn mapf, double* __restrict__ agg,
                                                     const int* gate) {
    extern __shared__ double sbuf[];
    if (gate && *((volatile const int*)gate) != 0) return;
    AMap<N> mine;
    block_scan<N, FWD, MapFn>(mapf, T, sbuf, mine);
    const int last = FWD ? AS_BLK - 1 : 0;
    if (threadIdx.x == last) amap_copy_to<N>(agg + (size_t)blockIdx.x * amap_doubles<N>(), mine);
}

// One CTA: entry state of every block.  FWD: entry(b) = Agg_{b-1} o ... o
// Agg_0 (s0).  BWD: entry(b) = Agg_{b+1} o ... o Agg_{nb-1} (eT), i.e. the
// state after the block's last step.  Hillis-Steele over the aggregates in
// global ping-pong buffers (nb <= 1024 blocks, T <= 131072 steps).
template <int N, bool FWD>
__global__ void __launch_bounds__(1024) affscan_k2(int nb, const double* __restrict__ init,
                                                   double* __restrict__ agg, double* __restrict__ tmp,
                                                   double* __restrict__ entry, const int* gate) {
    constexpr int AD = amap_doubles<N>();
    if (gate && *((volatile const int*)gate) != 0) return;
    const int t = threadIdx.x;
    double* cur = agg;
    double* nxt = tmp;
    for (int s = 1; s < nb; s <<= 1) {
        if (t < nb) {
            AMap<N> mine, other, res;
            amap_copy_from<N>(cur + (size_t)t * AD, mine);
            const int o = FWD ? t - s : t + s;
            if (o >= 0 && o < nb) {
                amap_copy_from<N>(cur + (size_t)o * AD, other);
                amap_compose<N>(mine, other, res);
                mine = res;
            }
            amap_copy_to<N>(nxt + (size_t)t * AD, mine);
        }
        __syncthreads();
        double* x = cur;
        cur = nxt;
        nxt = x;
    }
    if (t < nb) {
        double x0[N], y[N];
#pragma unroll
        for (int i = 0; i < N; ++i) x0[i] = init ? init[i] : 0.0;
        const int o = FWD ? t - 1 : t + 1;
        if (o >= 0 && o < nb) {
            AMap<N> a;
            amap_copy_from<N>(cur + (size_t)o * AD, a);
            amap_apply<N>(a, x0, y);
        } else {
#pragma unroll
            for (int i = 0; i < N; ++i) y[i] = x0[i];
        }
#pragma unroll
        for (int i = 0; i < N; ++i) entry[(size_t)t * N + i] = y[i];
    }
}

// Consumer: double operator()(int k, const double* before, const double* after)
//   FWD: before = s_k, after = s_{k+1};  BWD: before = e_{k+1}, after = e_k.
// Returns a value summed per block into red[blockIdx.x] (fixed order).
template <int N, bool FWD, class MapFn, class OutFn>
__global__ void __launch_bounds__(AS_BLK) affscan_k3(int T, MapFn mapf, OutFn out,
                                                     const double* __restrict__ entry,
                                                     double* __restrict__ red, const int* gate) {
    extern __shared__ double sbuf[];
    __shared__ double s_red[AS_BLK / 32];
    if (gate && *((volatile const int*)gate) != 0) return;
    constexpr int AD = amap_doubles<N>();
    AMap<N> mine;
    block_scan<N, FWD, MapFn>(mapf, T, sbuf, mine);
    // after the scan the last buffer written holds every thread's inclusive
    // map; the exclusive map of thread t is the inclusive one of t-1 (FWD) or
    // t+1 (BWD), identity at the block edge
    const int t = threadIdx.x;
    const int k = blockIdx.x * AS_BLK + t;
    const double* fin = sbuf + ((31 - __clz(AS_BLK)) % 2 == 0 ? 0 : AS_BLK * AD);
    double ein[N], before[N], after[N];
#pragma unroll
    for (int i = 0; i < N; ++i) ein[i] = entry[(size_t)blockIdx.x * N + i];
    amap_apply<N>(mine, ein, after);
    const int o = FWD ? t - 1 : t + 1;
    if (o >= 0 && o < AS_BLK) {
        AMap<N> ex;
        amap_copy_from<N>(fin + o * AD, ex);
        amap_apply<N>(ex, ein, before);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) before[i] = ein[i];
    }
    double v = 0.0;
    if (k < T) v = out(k, before, after);
    v = warp_sum(v);
    if ((t & 31) == 0) s_red[t >> 5] = v;
    __syncthreads();
    if (t == 0) {
        double s = 0.0;
        for (int w = 0; w < AS_BLK / 32; ++w) s += s_red[w];
        if (red) red[blockIdx.x] = s;
    }
}

template <int N>
inline size_t affscan_smem_bytes() {
    return 2 * AS_BLK * amap_doubles<N>() * sizeof(double);
}

inline int affscan_blocks(int T) { return (T + AS_BLK - 1) / AS_BLK; }

// scratch doubles: aggregates (2 x nb maps), entries (nb x N), block sums (nb)
template <int N>
inline size_t affscan_scratch_doubles(int T) {
    const size_t nb = affscan_blocks(T);
    return 2 * nb * amap_doubles<N>() + nb * N + nb;
}

struct AffScanBufs {
    double* agg;
    double* tmp;
    double* entry;
    double* red;
};

template <int N>
inline AffScanBufs affscan_bufs(double* scratch, int T) {
    const size_t nb = affscan_blocks(T);
    AffScanBufs b;
    b.agg = scratch;
    b.tmp = scratch + nb * amap_doubles<N>();
    b.entry = scratch + 2 * nb * amap_doubles<N>();
    b.red = b.entry + nb * N;
    return b;
}

// Launch the three kernels.  init: s_0 (FWD) / e_T (BWD) on device, or null
// for zeros.  Returns the number of launches.
template <int N, bool FWD, class MapFn, class OutFn>
inline int affscan_run(int T, const MapFn& mapf, const OutFn& out, const double* init,
                       const AffScanBufs& b, const int* gate, cudaStream_t st) {
    const int nb = affscan_blocks(T);
    const size_t smem = affscan_smem_bytes<N>();
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(affscan_k1<N, FWD, MapFn>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(affscan_k3<N, FWD, MapFn, OutFn>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    affscan_k1<N, FWD, MapFn><<<nb, AS_BLK, smem, st>>>(T, mapf, b.agg, gate);
    affscan_k2<N, FWD><<<1, 1024, 0, st>>>(nb, init, b.agg, b.tmp, b.entry, gate);
    affscan_k3<N, FWD, MapFn, OutFn><<<nb, AS_BLK, smem, st>>>(T, mapf, out, b.entry, b.red, gate);
    return 3;
}

}  // namespace fcb
