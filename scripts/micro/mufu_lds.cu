// MUFU.EX2 throughput with interleaved shared-memory loads (MIO contention).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

// per iteration: NL LDS.128 (stride: 1 = consecutive lanes, 0 = broadcast), 16 ex2
template <int NL, int BCAST>
__global__ void __launch_bounds__(512, 1) k(int iters, float seed, float* sink) {
    __shared__ float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i * 1e-6f, 1e-6f, 2e-6f, 3e-6f);
    __syncthreads();
    float a[16];
    for (int c = 0; c < 16; ++c) a[c] = seed * (threadIdx.x + c) * 1e-9f;
    float acc = 0.f;
    int base = BCAST ? 0 : (threadIdx.x & 31);
    for (int i = 0; i < iters; ++i) {
        const int off = (i * 64) & 2047;
        float4 v[NL > 0 ? NL : 1];
#pragma unroll
        for (int l = 0; l < NL; ++l) v[l] = s[(off + base + l * 32) & 2047];
#pragma unroll
        for (int c = 0; c < 16; ++c) a[c] = ex2(a[c]) * -1e-3f;
#pragma unroll
        for (int l = 0; l < NL; ++l) acc += v[l].x + v[l].w;
    }
    float t = acc;
    for (int c = 0; c < 16; ++c) t += a[c];
    if (t == 12345.f) *sink = t;
}

template <int NL, int B>
void run() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* sink; cudaMalloc(&sink, 4);
    int iters = 4000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<NL, B><<<sms, 512>>>(10, 1.f, sink);
    cudaEventRecord(e0);
    k<NL, B><<<sms, 512>>>(iters, 1.f, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ex = (double)sms * 512 * 16 * iters;
    printf("LDS.128/16ex2 %d %s: %.1f ex2/clk/SM\n", NL, B ? "broadcast" : "distinct ", ex / ms / 1e-3 / sms / 1.965e9);
}
int main() {
    run<0, 0>();
    run<2, 0>(); run<4, 0>(); run<6, 0>(); run<12, 0>();
    run<2, 1>(); run<6, 1>(); run<12, 1>();
    return 0;
}
