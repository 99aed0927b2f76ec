// fcb_internal.cuh -- shared device/host helpers for the flowcover-b200 kernels.
//
// Everything here is sm_100a-only: the library is compiled with
// -gencode arch=compute_100a,code=sm_100a and has no fallback path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <atomic>
#include <string>

#include "../../include/flowcover_b200.h"

namespace fcb {

// ---------------------------------------------------------------------------
// host-side status plumbing
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* where);
extern std::atomic<long long> g_launches;

extern std::atomic<const char*> g_last_kernel;

inline void count_launch(long long k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
inline void count_launch_named(const char* where) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    g_last_kernel.store(where, std::memory_order_relaxed);
}

#define FCB_CUDA(call)                                              \
    do {                                                            \
        cudaError_t _e = (call);                                    \
        if (_e != cudaSuccess) return ::fcb::cuda_status(_e, #call); \
    } while (0)

#define FCB_LAUNCHED(where)                                         \
    do {                                                            \
        ::fcb::count_launch_named(where);                           \
        cudaError_t _e = cudaGetLastError();                        \
        if (_e != cudaSuccess) return ::fcb::cuda_status(_e, where); \
    } while (0)

int sm_count();          // cached per current device
int current_device();

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Arena {
    char* base;
    size_t cap;
    size_t off = 0;
    bool ok = true;
    Arena(void* p, size_t n) : base(static_cast<char*>(p)), cap(n) {}
    template <typename T>
    T* take(size_t count) {
        size_t o = align_up(off, 256);
        size_t bytes = count * sizeof(T);
        if (base == nullptr) {  // sizing pass
            off = o + bytes;
            return nullptr;
        }
        if (o + bytes > cap) {
            ok = false;
            off = o + bytes;
            return nullptr;
        }
        off = o + bytes;
        return reinterpret_cast<T*>(base + o);
    }
};

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
constexpr double kLog2e = 1.4426950408889634073599;

// scal[] layout of a transport solve (device double[16]; fcb_resolve_omega)
enum { SC_OMEGA = 0, SC_S = 1, SC_C = 2 /*2..4*/, SC_MX2 = 5, SC_MX = 6 /*6..8*/, SC_MY2 = 9,
       SC_MY = 10 /*10..12*/ };
constexpr double kLn2 = 0.6931471805599453094172;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x for two lanes on the FMA pipe instead of the MUFU (XU) pipe, for sweeps
// whose MUFU.EX2 rate is the bound and whose issue slots have headroom: the
// argument is clamped to [-125, 127], split x = j + f with j = rint(x) by the
// 1.5*2^23 rounding constant, 2^f (|f| <= 1/2) from a degree-5 relative-error
// minimax polynomial (max rel. error 2.4e-7 in fp32 Horner, the same order as
// ex2.approx), and j is added into the exponent field.  Below -125 the result
// is ~2^-125 instead of ex2.approx.ftz's 0 (terms are summed with >= 1);
// above 127 it is ~2^127 (the sweep's out-of-range test still fires).
// 14 issue slots for two values vs 2 MUFU instructions (8 XU cycles each).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x.x = fminf(fmaxf(x.x, -125.f), 127.f);
    x.y = fminf(fmaxf(x.y, -125.f), 127.f);
    const float2 rnd = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
    const float2 j = __fadd2_rn(x, rnd);                     // rint(x) in the low bits
    const float2 jf = __fadd2_rn(j, make_float2(-12582912.f, -12582912.f));
    const float2 f = __ffma2_rn(jf, make_float2(-1.f, -1.f), x);  // exact, |f| <= 1/2
    float2 p = __ffma2_rn(make_float2(1.32764654699713e-3f, 1.32764654699713e-3f), f,
                          make_float2(9.675540961325169e-3f, 9.675540961325169e-3f));
    p = __ffma2_rn(p, f, make_float2(5.550713464617729e-2f, 5.550713464617729e-2f));
    p = __ffma2_rn(p, f, make_float2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
    p = __ffma2_rn(p, f, make_float2(6.931469440460205e-1f, 6.931469440460205e-1f));
    p = __ffma2_rn(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
    // bits(j) = bits(1.5 * 2^23) + j, and bits(1.5 * 2^23) << 23 == 0 (mod 2^32)
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}

template <typename T> struct Vec4;
template <> struct alignas(16) Vec4<float> { float x, y, z, w; };
template <> struct alignas(32) Vec4<double> { double x, y, z, w; };

__device__ __forceinline__ float vget(const Vec4<float>& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : v.z);
}
__device__ __forceinline__ double vget(const Vec4<double>& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : v.z);
}

// Arithmetic traits: float works in log2 units with MUFU.EX2, double in
// natural units with the IEEE-accurate exp/log.
template <typename Real> struct Units;
template <> struct Units<float> {
    static constexpr double unit = kLog2e;   // exponent units per natural unit
    __device__ static __forceinline__ float expu(float x) { return ex2_approx(x); }
    __device__ static __forceinline__ double logu(double x) { return log2(x); }
};
template <> struct Units<double> {
    static constexpr double unit = 1.0;
    __device__ static __forceinline__ double expu(double x) { return exp(x); }
    __device__ static __forceinline__ double logu(double x) { return log(x); }
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier for cooperatively launched kernels: one arrival counter
// that only grows (the caller zeroes it before the launch).  Barrier k of the
// launch completes when the counter reaches k * nblocks, so a CTA derives its
// target from the value its own arrival returned -- no generation word, no
// reset, one atomic per CTA.  Measured 1.36 us per barrier at 296 CTAs
// against 2.4 us for a count/generation pair with full fences.
struct GridBarrier {
    unsigned long long count;  // arrivals; 64-bit so it cannot wrap within a launch
    unsigned pad[30];   // own 128-byte line
    unsigned work;      // dynamic work-item counter (grows across phases)
    unsigned pad2[31];
};

#ifdef FCB_TIMELINE
// Debug builds only (scripts/tune_ot.sh -DFCB_TIMELINE): block 0 records the
// globaltimer when it arrives at and leaves every grid barrier.
__device__ unsigned long long g_timeline[8192];
__device__ unsigned g_timeline_n;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define FCB_TL_MARK()                                                          \
    do {                                                                       \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                             \
            unsigned i_ = g_timeline_n;                                        \
            if (i_ < 8192) g_timeline[i_] = gtimer();                          \
            g_timeline_n = i_ + 1;                                             \
        }                                                                      \
    } while (0)
#else
#define FCB_TL_MARK() \
    do {              \
    } while (0)
#endif

__device__ __forceinline__ void grid_sync(GridBarrier* b) {
    __syncthreads();
    FCB_TL_MARK();
    if (threadIdx.x == 0) {
        const unsigned long long nb = gridDim.x * gridDim.y * gridDim.z;
        // the CTA's writes (ordered before this thread by bar.sync) are
        // released at gpu scope before the arrival
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const unsigned long long old = atomicAdd(&b->count, 1ull);
        const unsigned long long target = (old / nb + 1ull) * nb;
        while (ld_acquire_u64(&b->count) < target) __nanosleep(20);
    }
    __syncthreads();
    FCB_TL_MARK();
}

// max over non-negative doubles (NaN propagates: its bit pattern sorts above +inf)
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* slot, double v) {
    atomicMax(slot, static_cast<unsigned long long>(__double_as_longlong(v)));
}

__device__ __forceinline__ double load_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ float load_cg(const float* p) { return __ldcg(p); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block-wide sum (fixed tree); result valid in thread 0.
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = (threadIdx.x < BLOCK / 32) ? scratch[threadIdx.x] : 0.0;
        r = warp_sum(r);
    }
    return r;
}

}  // namespace fcb
