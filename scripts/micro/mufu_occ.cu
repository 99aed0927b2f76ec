// MUFU.EX2 throughput vs resident warps and interleaved FP32 work.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_occ mufu_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int CH, int FMA2>
__global__ void k(int iters, float seed, float* sink) {
    float a[CH];
    float2 acc = make_float2(0.f, 0.f);
    for (int c = 0; c < CH; ++c) a[c] = seed * (threadIdx.x + c) * 1e-9f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; c += 2) {
            float e0 = ex2(a[c]), e1 = ex2(a[c + 1]);
#pragma unroll
            for (int f = 0; f < FMA2; ++f) acc = __ffma2_rn(make_float2(e0, e1), make_float2(1.0001f, 0.9999f), acc);
            a[c] = e0 * -1e-3f; a[c + 1] = e1 * -1e-3f;
        }
    }
    float s = acc.x + acc.y;
    for (int c = 0; c < CH; ++c) s += a[c];
    if (s == 12345.f) *sink = s;
}

template <int CH, int FMA2>
void run(int blocks_per_sm, int threads) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* sink; cudaMalloc(&sink, 4);
    int iters = 2000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<CH, FMA2><<<sms * blocks_per_sm, threads>>>(10, 1.f, sink);
    cudaEventRecord(e0);
    k<CH, FMA2><<<sms * blocks_per_sm, threads>>>(iters, 1.f, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ex = (double)sms * blocks_per_sm * threads * CH * iters;
    printf("warps/SM %3d chains %2d ffma2/ex2pair %d : %.3f Tex2/s = %.1f /clk/SM @1.965GHz\n",
           blocks_per_sm * threads / 32, CH, FMA2, ex / ms / 1e9, ex / ms / 1e-3 / sms / 1.965e9);
    cudaFree(sink);
}
int main() {
    run<8, 0>(8, 256);
    run<8, 0>(1, 512);
    run<16, 0>(1, 512);
    run<32, 0>(1, 512);
    run<8, 0>(1, 256);
    run<16, 0>(1, 256);
    run<16, 2>(1, 512);
    run<16, 4>(1, 512);
    run<16, 6>(1, 512);
    run<16, 4>(2, 512);
    return 0;
}
