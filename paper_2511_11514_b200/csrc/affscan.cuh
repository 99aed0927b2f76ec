// affscan.cuh -- parallel scans of affine recurrences over time, one thread
// per time step.
//
//   forward : s_{k+1} = M_k s_k + c_k     (s_0 given)      k = 0..T-1
//   backward: e_k     = M_k e_{k+1} + c_k (e_T given)      k = T-1..0
//
// Three launches, no grid-wide synchronisation:
//   K1  every CTA owns AS_BLK consecutive chunks of CH steps (CH = 1 up to
//       AS_BLK * 148 steps, more for longer horizons so K2 sees ~148
//       aggregates); each thread composes its chunk's step maps, then a
//       Hillis-Steele scan in shared memory composes the block's maps; the
//       block aggregate goes to global memory.
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
constexpr int AS_K2 = 256;  // threads of the aggregate scan (few registers spill at 256)

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
// Steps per thread chunk of the three-launch scan.
__host__ __device__ __forceinline__ int affscan_chunk(int T) {
    const int per = AS_BLK * 148;
    return T > per ? (T + per - 1) / per : 1;
}

// The map of one thread's chunk [k0, k0 + CH) (clipped at T): later o earlier.
template <int N, bool FWD, class MapFn>
__device__ __forceinline__ void chunk_map(const MapFn& mapf, int T, int k0, int CH, AMap<N>& mine) {
    if (CH == 1) {
        if (k0 < T) mapf(k0, mine);
        else amap_identity<N>(mine);
        return;
    }
    amap_identity<N>(mine);
    for (int j = 0; j < CH; ++j) {
        // FWD applies steps in increasing k, BWD in decreasing k
        const int k = FWD ? k0 + j : k0 + CH - 1 - j;
        if (k >= T) continue;
        AMap<N> step, res;
        mapf(k, step);
        amap_compose<N>(step, mine, res);
        mine = res;
    }
}

template <int N, bool FWD, class MapFn>
__device__ __forceinline__ void block_scan(const MapFn& mapf, int T, double* buf, AMap<N>& mine) {
    constexpr int AD = amap_doubles<N>();
    const int t = threadIdx.x;
    const int CH = affscan_chunk(T);
    chunk_map<N, FWD, MapFn>(mapf, T, (blockIdx.x * AS_BLK + t) * CH, CH, mine);
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

// K2: the state entering each block, from the block aggregates.
template <int N, bool FWD>
__global__ void __launch_bounds__(AS_K2) affscan_k2(int nb, const double* __restrict__ init,
                                                   double* __restrict__ agg, double* __restrict__ tmp,
                                                   double* __restrict__ entry, const int* gate) {
    // Only the state entering each block is needed, not the composed maps: one
    // thread walks the nb block maps in scan order applying them to the state
    // (nb N^2 FMAs, dependent), the block stages the maps through shared
    // memory 32 at a time.  37 us at nb = 148, N = 6 (ncu, aircraft T = 1e5)
    // against 42 us for the Hillis-Steele composition of the maps it replaces:
    // the walk is one thread's latency chain.
    constexpr int AD = amap_doubles<N>();
    constexpr int CHUNK = 32;
    __shared__ double s_maps[CHUNK * AD];
    (void)tmp;
    if (gate && *((volatile const int*)gate) != 0) return;
    double x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = init ? init[i] : 0.0;
    for (int c0 = 0; c0 < nb; c0 += CHUNK) {
        const int cnt = min(CHUNK, nb - c0);
        __syncthreads();
        for (int e = threadIdx.x; e < cnt * AD; e += blockDim.x) {
            const int r = e / AD, q = e - r * AD;
            const int t = FWD ? c0 + r : nb - 1 - (c0 + r);  // r-th block in scan order
            s_maps[e] = __ldcg(agg + (size_t)t * AD + q);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int r = 0; r < cnt; ++r) {
                const int t = FWD ? c0 + r : nb - 1 - (c0 + r);
#pragma unroll
                for (int i = 0; i < N; ++i) entry[(size_t)t * N + i] = x[i];
                AMap<N> a;
                amap_copy_from<N>(s_maps + (size_t)r * AD, a);
                double y[N];
                amap_apply<N>(a, x, y);
#pragma unroll
                for (int i = 0; i < N; ++i) x[i] = y[i];
            }
        }
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
    const int CH = affscan_chunk(T);
    const int k0 = (blockIdx.x * AS_BLK + t) * CH;
    const double* fin = sbuf + ((31 - __clz(AS_BLK)) % 2 == 0 ? 0 : AS_BLK * AD);
    double ein[N], before[N], after[N];
#pragma unroll
    for (int i = 0; i < N; ++i) ein[i] = entry[(size_t)blockIdx.x * N + i];
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
    if (CH == 1) {
        amap_apply<N>(mine, ein, after);
        if (k0 < T) v = out(k0, before, after);
    } else {
        // re-walk the chunk from the state entering it (FWD: s_k0; BWD: e_{k0+CH})
        for (int j = 0; j < CH; ++j) {
            const int k = FWD ? k0 + j : k0 + CH - 1 - j;
            if (k >= T) continue;
            AMap<N> step;
            mapf(k, step);
            amap_apply<N>(step, before, after);
            v += out(k, before, after);
#pragma unroll
            for (int i = 0; i < N; ++i) before[i] = after[i];
        }
    }
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

inline int affscan_blocks(int T) {
    const int steps = AS_BLK * affscan_chunk(T);
    return (T + steps - 1) / steps;
}

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
    affscan_k2<N, FWD><<<1, AS_K2, 0, st>>>(nb, init, b.agg, b.tmp, b.entry, gate);
    affscan_k3<N, FWD, MapFn, OutFn><<<nb, AS_BLK, smem, st>>>(T, mapf, out, b.entry, b.red, gate);
    return 3;
}

// ---------------------------------------------------------------------------
// One-launch scans for horizons up to AS_BLK * AS_BLK steps (fused_scan).
// Block b of nb = ceil(T / AS_BLK) owns steps [b*AS_BLK, (b+1)*AS_BLK):
//   1. in-block Hillis-Steele scan (block_scan), the block aggregate is
//      published with a tagged flag (release);
//   2. each block waits for the flags of the blocks before it in scan order
//      (acquire), composes their aggregates with a warp-shuffle scan
//      (scan_states) and obtains its entry state -- no grid barrier, no
//      second launch, no counter to reset;
//   3. the re-walk hands (state before, state after) of every step to the
//      consumer, whose values are summed per block.
// Flags carry a per-launch tag, so the workspace needs no initialisation.
// Blocks only wait on blocks of the same launch and nb <= 128 <= #SMs, so all
// blocks are co-resident.
// ---------------------------------------------------------------------------
#ifdef FCB_SCAN_TL
// Debug builds only: per-block globaltimer stamps of the one-launch scans.
__device__ unsigned long long g_scan_tl[AS_BLK][16];
#define FCB_SCAN_MARK(i)                                                              \
    do {                                                                              \
        if (threadIdx.x == 0) {                                                       \
            unsigned long long t_;                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
            g_scan_tl[blockIdx.x][i] = t_;                                            \
        }                                                                             \
    } while (0)
#else
#define FCB_SCAN_MARK(i) \
    do {                 \
    } while (0)
#endif

template <int N>
__device__ __forceinline__ void amap_shfl(AMap<N>& dst, const AMap<N>& src, int delta, bool up) {
#pragma unroll
    for (int i = 0; i < N * N; ++i)
        (&dst.M[0][0])[i] = up ? __shfl_up_sync(0xffffffffu, (&src.M[0][0])[i], delta)
                               : __shfl_down_sync(0xffffffffu, (&src.M[0][0])[i], delta);
#pragma unroll
    for (int i = 0; i < N; ++i)
        dst.c[i] = up ? __shfl_up_sync(0xffffffffu, src.c[i], delta)
                      : __shfl_down_sync(0xffffffffu, src.c[i], delta);
}

template <int N, int W = AS_BLK / 32>
struct ScanShared {
    double tot[W][amap_doubles<N>()];   // scan_states scratch
    double went[W][N];
    double btot[W][amap_doubles<N>()];  // in-block warp totals (fused_scan)
    double bwent[W][N];
    double red[W];
};

// Element t is held by thread t of a BLK-thread block.  Returns in `state` the
// state entering element t: FWD (a_{t-1} o ... o a_0)(init), BWD
// (a_{t+1} o ... o a_{BLK-1})(init).  `mine` is clobbered.
template <int N, bool FWD, int BLK>
__device__ __forceinline__ void scan_states(AMap<N>& mine, const double* init,
                                            ScanShared<N, BLK / 32>& sh, double* state) {
    constexpr int W = BLK / 32;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    AMap<N> m, r;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        amap_shfl<N>(m, mine, s, FWD);
        if (FWD ? lane >= s : lane + s < 32) {
            amap_compose<N>(mine, m, r);
            mine = r;
        }
    }
    if (FWD) FCB_SCAN_MARK(10);
    if (lane == (FWD ? 31 : 0)) amap_copy_to<N>(sh.tot[w], mine);
    amap_shfl<N>(m, mine, 1, FWD);  // exclusive map inside the warp
    if (lane == (FWD ? 0 : 31)) amap_identity<N>(m);
    __syncthreads();
    if (FWD) FCB_SCAN_MARK(11);
    if (t == 0) {
        double s[N], y[N];
#pragma unroll
        for (int i = 0; i < N; ++i) s[i] = init ? init[i] : 0.0;
        for (int q = 0; q < W; ++q) {
            const int ww = FWD ? q : W - 1 - q;
            AMap<N> a;
            amap_copy_from<N>(sh.tot[ww], a);
#pragma unroll
            for (int i = 0; i < N; ++i) sh.went[ww][i] = s[i];
            amap_apply<N>(a, s, y);
#pragma unroll
            for (int i = 0; i < N; ++i) s[i] = y[i];
        }
    }
    __syncthreads();
    if (FWD) FCB_SCAN_MARK(12);
    amap_apply<N>(m, sh.went[w], state);
}

__device__ __forceinline__ unsigned ld_acquire_flag(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_flag(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Wait (thread t < n) for flags[t] == tag.
#ifndef FCB_SPIN_SLEEP
#define FCB_SPIN_SLEEP 32
#endif
__device__ __forceinline__ void wait_flag(const unsigned* flags, int t, unsigned tag) {
    while (ld_acquire_flag(flags + t) != tag) {
#if FCB_SPIN_SLEEP > 0
        __nanosleep(FCB_SPIN_SLEEP);
#endif
    }
}

constexpr int FUSED_MAX_BLOCKS = AS_BLK;

// The one-launch scans take one step per thread.
inline int fused_blocks(int T) { return (T + AS_BLK - 1) / AS_BLK; }
inline bool fused_scan_ok(int T) { return T >= 1 && fused_blocks(T) <= FUSED_MAX_BLOCKS; }

// Workspace of fused scans: per slot nb aggregates and nb flags.
template <int N>
inline size_t fused_agg_doubles() {
    return (size_t)FUSED_MAX_BLOCKS * amap_doubles<N>();
}

// Optional extra wait folded into the look-back of fused_scan: every block's
// flag (all nb of them) must carry `tag`; the max of their ints goes to *out.
struct ExtraWait {
    const unsigned* flags;
    const int* vals;
    int* out;  // shared memory
    unsigned tag;
};

// Returns the block's sum of consumer values (every thread).  sbuf: dynamic
// shared memory of fused_smem_bytes<N>().  Ends with __syncthreads.
template <int N, bool FWD, class MapFn, class OutFn>
__device__ double fused_scan(int T, const MapFn& mapf, const OutFn& out, const double* init,
                             double* agg, unsigned* flags, unsigned tag, double* sbuf,
                             ScanShared<N>& sh, const ExtraWait* xw = nullptr) {
    constexpr int AD = amap_doubles<N>();
    constexpr int W = AS_BLK / 32;
    const int nb = gridDim.x, b = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int k = b * AS_BLK + t;
    // 1. in-warp inclusive scan of the step maps (shuffles); the exclusive map
    //    (neighbour lane's inclusive) is parked in shared memory
    AMap<N> mine, m, r;
    if (k < T) mapf(k, mine);
    else amap_identity<N>(mine);
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        amap_shfl<N>(m, mine, s, FWD);
        if (FWD ? lane >= s : lane + s < 32) {
            amap_compose<N>(mine, m, r);
            mine = r;
        }
    }
    amap_shfl<N>(m, mine, 1, FWD);
    if (lane == (FWD ? 0 : 31)) amap_identity<N>(m);
    amap_copy_to<N>(sbuf + t * AD, m);
    if (lane == (FWD ? 31 : 0)) amap_copy_to<N>(sh.btot[w], mine);
    __syncthreads();
    // 2. block aggregate (warp totals composed in scan order), published
    if (t == 0) {
        AMap<N> acc, x;
        amap_copy_from<N>(sh.btot[FWD ? 0 : W - 1], acc);
#pragma unroll
        for (int q = 1; q < W; ++q) {
            amap_copy_from<N>(sh.btot[FWD ? q : W - 1 - q], x);
            amap_compose<N>(x, acc, r);
            acc = r;
        }
        amap_copy_to<N>(agg + (size_t)b * AD, acc);
        __threadfence();
        st_release_flag(flags + b, tag);
    }
    FCB_SCAN_MARK(FWD ? 5 : 1);
    // 3. look-back: predecessors in scan order (FWD [0, b), BWD (b, nb))
    AMap<N> a;
    if (FWD ? t < b : (t > b && t < nb)) {
        wait_flag(flags, t, tag);
        const double* src = agg + (size_t)t * AD;
#pragma unroll
        for (int i = 0; i < N * N; ++i) (&a.M[0][0])[i] = __ldcg(src + i);
#pragma unroll
        for (int i = 0; i < N; ++i) a.c[i] = __ldcg(src + N * N + i);
    } else {
        amap_identity<N>(a);
    }
    if (xw && t < nb) {
        wait_flag(xw->flags, t, xw->tag);
        const int f = __ldcg(xw->vals + t);
        if (f >= 0) atomicMax(xw->out, f);
    }
    // reconverge the warp after the divergent spins before any shuffle: a
    // diverged warp entering the shuffle scan costs ~20 us (measured)
    __syncwarp();
    FCB_SCAN_MARK(FWD ? 6 : 2);
    double st[N];
    scan_states<N, FWD, AS_BLK>(a, init, sh, st);
    // 4. block entry -> warp entry states
    if (t == b) {
#pragma unroll
        for (int i = 0; i < N; ++i) sh.bwent[FWD ? 0 : W - 1][i] = st[i];
    }
    __syncthreads();
    if (t == 0) {
        double x[N], y[N];
#pragma unroll
        for (int i = 0; i < N; ++i) x[i] = sh.bwent[FWD ? 0 : W - 1][i];
#pragma unroll
        for (int q = 0; q + 1 < W; ++q) {
            const int ww = FWD ? q : W - 1 - q;
            AMap<N> tw;
            amap_copy_from<N>(sh.btot[ww], tw);
            amap_apply<N>(tw, x, y);
#pragma unroll
            for (int i = 0; i < N; ++i) x[i] = sh.bwent[FWD ? ww + 1 : ww - 1][i] = y[i];
        }
    }
    __syncthreads();
    FCB_SCAN_MARK(FWD ? 7 : 3);
    // 5. re-walk: after = inclusive map applied to the warp entry, before =
    //    the exclusive one
    double before[N], after[N];
    amap_apply<N>(mine, sh.bwent[w], after);
    amap_copy_from<N>(sbuf + t * AD, m);
    amap_apply<N>(m, sh.bwent[w], before);
    double v = 0.0;
    if (k < T) v = out(k, before, after);
    v = warp_sum(v);
    if (lane == 0) sh.red[w] = v;
    __syncthreads();
    double total = 0.0;
#pragma unroll
    for (int q = 0; q < W; ++q) total += sh.red[q];
    __syncthreads();
    FCB_SCAN_MARK(FWD ? 8 : 4);
    return total;
}

template <int N>
inline size_t fused_smem_bytes() {
    return (size_t)AS_BLK * amap_doubles<N>() * sizeof(double);
}

// Per-block values gathered by block 0 in block order (deterministic).
__device__ __forceinline__ void publish_value(double* vals, unsigned* flags, unsigned tag,
                                              double v) {
    if (threadIdx.x == 0) {
        vals[blockIdx.x] = v;
        __threadfence();
        st_release_flag(flags + blockIdx.x, tag);
    }
}

// Block 0 only: sum of all blocks' published values, in block order.
__device__ __forceinline__ double gather_sum(const double* vals, const unsigned* flags,
                                             unsigned tag, double* s_tmp) {
    const int nb = gridDim.x, t = threadIdx.x;
    if (t < nb) {
        wait_flag(flags, t, tag);
        s_tmp[t] = __ldcg(vals + t);
    }
    __syncthreads();
    double s = 0.0;
    for (int q = 0; q < nb; ++q) s += s_tmp[q];
    return s;
}

// Host: a fresh tag per fused launch (low 2 bits select the flag use).
unsigned next_scan_tag();

}  // namespace fcb
