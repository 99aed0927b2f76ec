// flow_resident.cu -- host entry points of the shared-memory resident
// Sinkhorn flow (device code: flow_resident.cuh).
#include "flow_resident.cuh"

namespace fcb {

// Epochs of grid-group launches (shared by every kernel that uses RsArgs'
// barrier): odd, never repeating within ~2^31 launches.
unsigned next_launch_epoch() {
    static std::atomic<unsigned> launches{0};
    return 0x9e3779b9u * (launches.fetch_add(1u) + 1u) | 1u;
}

template <int D, bool GRID>
__global__ void __launch_bounds__(RS_BLOCK, 1) rs_flow_kernel(RsArgs A) {
    if (GRID) rs_start_epoch(A);
    rs_flow_body<D, GRID>(A, true);
}

bool sinkhorn_flow_resident_fits(int n, int m, int d) {
    if (const char* e = getenv("FCB_RESIDENT")) {
        if (e[0] == '0') return false;
    }
    if (d < 1 || d > 3 || n < 1 || m < 1) return false;
    return rs_shape(n, m, d, sm_count()).ok;
}

size_t sinkhorn_flow_resident_ws_bytes(int n, int m, int d) {
    return rs_layout(1, n, m, d, sm_count(), nullptr, 0).total;
}

template <int D, bool GRID>
static int rs_launch(RsArgs& a, int grid, size_t smem, cudaStream_t st) {
    auto kern = rs_flow_kernel<D, GRID>;
    static size_t attr_bytes = 0;
    if (attr_bytes < smem) {
        FCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_bytes = smem;
    }
    if (GRID) {
        void* args[] = {&a};
        FCB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(RS_BLOCK), args,
                                             smem, st));
    } else {
        kern<<<grid, RS_BLOCK, smem, st>>>(a);
    }
    FCB_LAUNCHED("rs_flow_kernel");
    return FCB_OK;
}


int sinkhorn_flow_resident(const double* X, int n, const double* Y, int m, int d,
                           double omega_fixed, int max_iters, double tol, double* warm_f,
                           double* warm_p, int* warm_valid, double* flow, double* fstat,
                           int* plan_state, int iteration, double* flow_log, double conv_tol,
                           void* ws, size_t ws_bytes, cudaStream_t st) {
    const int G = sm_count();
    const RsShape sh = rs_shape(n, m, d, G);
    if (!sh.ok) return fail(FCB_ENOTSUP, "point sets do not fit in shared memory");
    RsWs L = rs_layout(1, n, m, d, G, ws, ws_bytes);
    if (L.total > ws_bytes) return fail(FCB_EWORKSPACE, "sinkhorn_flow workspace too small");
    RsArgs a{};
    a.X = X;
    a.Y = Y;
    a.n = n;
    a.m = m;
    a.omega_fixed = omega_fixed;
    a.max_iters = max_iters;
    a.tol = tol;
    a.conv_tol = conv_tol;
    a.warm_f = warm_f;
    a.warm_p = warm_p;
    a.warm_valid = (warm_f && warm_p) ? warm_valid : nullptr;
    a.flow = flow;
    a.fstat = fstat;
    a.plan_state = plan_state;
    a.iteration = iteration;
    a.flow_log = flow_log;
    a.log_stride = 0;
    rs_fill(a, L, sh);
    if (getenv("FCB_RS_VERBOSE"))
        fprintf(stderr, "rs_flow: n=%d m=%d d=%d G=%d plan A=%d/%d B=%d/%d S=%d/%d smem=%zu\n", n, m,
                d, G, 1 << sh.A.cg, sh.A.nr, 1 << sh.B.cg, sh.B.nr, 1 << sh.S.cg, sh.S.nr, sh.smem);
    a.launch_id = next_launch_epoch();
    switch (d) {
        case 1: return rs_launch<1, true>(a, G, sh.smem, st);
        case 2: return rs_launch<2, true>(a, G, sh.smem, st);
        default: return rs_launch<3, true>(a, G, sh.smem, st);
    }
}

extern "C" FCB_API long long fcb_debug_careful_rows_resident(void) {
    unsigned v = 0, zero = 0;
    if (cudaMemcpyFromSymbol(&v, g_rs_careful_rows, sizeof(unsigned)) != cudaSuccess) return -1;
    cudaMemcpyToSymbol(g_rs_careful_rows, &zero, sizeof(unsigned));
    return (long long)v;
}

extern "C" FCB_API int fcb_debug_rs_timeline(unsigned long long* host_out, int cap) {
#ifdef FCB_TIMELINE
    unsigned n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, g_rs_tl_n, sizeof(unsigned));
    const int k = (int)std::min<unsigned>(n, (unsigned)cap);
    if (k) cudaMemcpyFromSymbol(host_out, g_rs_tl, k * sizeof(unsigned long long));
    const unsigned zero = 0;
    cudaMemcpyToSymbol(g_rs_tl_n, &zero, sizeof(unsigned));
    return k;
#else
    (void)host_out;
    (void)cap;
    return -1;
#endif
}

}  // namespace fcb
