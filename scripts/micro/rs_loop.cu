// Throughput of the resident sweep's pair loop (rs_rows) in isolation:
// one CTA of 512 threads per SM, synthetic columns in shared memory.
// nvcc ... -I../../paper_2511_11514_b200/csrc rs_loop.cu
#include "../../paper_2511_11514_b200/csrc/flow_resident.cu"
#include <cstdio>

namespace fcb {
struct SynthRows {
    __device__ __forceinline__ double rowc2(int li) const { return -1.0 * li; }
    __device__ __forceinline__ void init(int li, float* x, float& rc) const {
        x[0] = 0.01f * (li % 7);
        x[1] = 0.02f * (li % 5);
        if (3 > 2) {}
        rc = -2.0f;
    }
};

template <int NR, bool BARY>
__global__ void __launch_bounds__(RS_BLOCK, 1) loop_kernel(int cols, int cg, int reps, float* out) {
    __shared__ RsRes res[RS_BLOCK];
    __shared__ RsRes xw[RS_WARPS * 8];
    RsCols c;
    const int nq = (cols + 3) / 4;
    const int nqp = (nq + (2 << cg) - 1) / (2 << cg) * (2 << cg);
    c.q[0] = 0; c.q[1] = 4 * nqp; c.q[2] = 0; c.w = 8 * nqp; c.nq = nq; c.nqp = nqp;
    for (int j = threadIdx.x; j < 4 * nqp; j += RS_BLOCK) {
        rs_smem[c.q[0] + j] = 0.001f * (j % 13);
        rs_smem[c.q[1] + j] = 0.002f * (j % 11);
        rs_smem[c.w + j] = j < cols ? -0.5f - 0.01f * (j % 17) : -INFINITY;
    }
    __syncthreads();
    const int RG = RS_BLOCK >> cg;
    RsPassMap pm{0, NR, 0, NR};
    (void)RG;
    for (int r = 0; r < reps; ++r) {
        rs_rows<2, NR, BARY>(c, cg, pm, SynthRows{}, res, xw);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = res[0].s;
}
}  // namespace fcb

template <int NR, bool BARY>
void run(int cols, int cg) {
    using namespace fcb;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; cudaMalloc(&out, sms * 4);
    const int nq = (cols + 3) / 4;
    const int nqp = (nq + (2 << cg) - 1) / (2 << cg) * (2 << cg);
    size_t smem = 12 * nqp * 4;
    cudaFuncSetAttribute(loop_kernel<NR, BARY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 20;
    loop_kernel<NR, BARY><<<sms, RS_BLOCK, smem>>>(cols, cg, 2, out);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    loop_kernel<NR, BARY><<<sms, RS_BLOCK, smem>>>(cols, cg, reps, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double rows = (double)(RS_BLOCK >> cg) * NR;
    const double pairs = (double)sms * reps * rows * 4.0 * nqp;
    printf("NR %d BARY %d CG %3d cols %6d: %.2f pairs/clk/SM (%.1f%% of MUFU) err=%s\n", NR, (int)BARY, 1 << cg, cols,
           pairs / (ms * 1e-3) / sms / 1.965e9, 100.0 * pairs / (ms * 1e-3) / sms / 1.965e9 / 16.0,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run<1, false>(2000, 5); run<2, false>(2000, 5); run<4, false>(2000, 5); run<6, false>(2000, 5);
    run<1, true>(10000, 6); run<2, true>(10000, 6); run<4, true>(10000, 7); run<3, true>(10000, 7);
    run<4, false>(10000, 7); run<2, true>(10000, 5); run<4, true>(10000, 5);
    return 0;
}
