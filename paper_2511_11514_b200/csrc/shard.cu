// shard.cu -- device steps of the M-sharded flows (BASELINE config 4).
//
// One process per GPU; the reference samples Y (Sinkhorn) or the SVGD sources
// are split across ranks.  The host (paper_2511_11514_b200/distributed.py)
// strings these kernels together with NCCL collectives on the same stream, so
// an inner iteration never waits for the host:
//
//   Sinkhorn cross solve (_solve_asymmetric, sinkhorn.py:170-205), rank r:
//     g_r = w (log b - LSE(Y_r vs X; f))          fcb_lse_sweep   (local)
//     {L_r, ybar_r} = LSE(X vs Y_r; g_r)           fcb_lse_sweep   (local)
//     all_gather {L_r, ybar_r}                     NCCL
//     merge in fixed rank order -> f_new, err      fcb_shard_cross_merge
//   Self term (_solve_symmetric, sinkhorn.py:208-236), rows of X sharded:
//     {L, xbar} of own rows vs all X; p_new, ...   fcb_lse_sweep + fcb_shard_self_rows
//     all_gather own rows                          NCCL
//     err, commit p                                fcb_shard_self_commit
//   then the envelope gradient, FlowError test, warm state and planner hooks
//   (sinkhorn.py:370-397)                          fcb_shard_flow_finish
//
// Loop control lives in a device word per solve (done flag, iteration count):
// the host queues iterations ahead and every kernel of a finished solve is a
// no-op.  Collectives of such iterations re-send unchanged buffers.  Merges use
// a fixed rank order and decisions are taken on replicated values, so every
// rank holds bit-identical potentials and takes the same branch.
//
//   SVGD (stein.py:79-122), sources sharded: each rank sums k_ij and
//   k_ij (s_j - (2/h) x_j) over its own sources j for every query i
//   (fcb_stein_partial), the partials are all-gathered and summed in rank
//   order (fcb_stein_combine), which also runs the planner hooks.
#include <algorithm>

#include "fcb_internal.cuh"

namespace fcb {

int lse_sweep(int precision, const double* R, int nr, const double* S, int ns, int d,
              const double* scal, const double* pot, const double* row_est, double row_logw,
              double out_scale, double out_shift, double* out, double* bary, const int* gate,
              void* ws, size_t ws_bytes, cudaStream_t st);
size_t ot_ws_bytes(int mode, int precision, int n, int m, int d);

constexpr int SH_BLOCK = 256;
constexpr int SH_ONE = 1024;
constexpr double SH_EXP_CLIP = 500.0;         // sinkhorn.py:67
constexpr double SH_OMEGA_FLOOR = 1e-12;      // sinkhorn.py:66
constexpr double SH_AUTO_OMEGA = 0.05;        // sinkhorn.py:65

// ctl[] words of one sharded flow
enum { CTL_DONE_X = 0, CTL_DONE_P = 1, CTL_IT_X = 2, CTL_IT_P = 3, CTL_CNT_X = 4, CTL_CNT_P = 5,
       CTL_CNT_F = 6, CTL_SKIP = 7 };

static int sh_blocks(long n) {
    return (int)std::max<long>(1, std::min<long>(4L * sm_count(), (n + SH_BLOCK - 1) / SH_BLOCK));
}

// ---------------------------------------------------------------------------
// point sums: out = {sum_k p_ik (d), sum |p_i|^2, n}; one block, fixed order
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SH_ONE) point_sums_kernel(const double* __restrict__ P, int n,
                                                            int d, double* __restrict__ out) {
    __shared__ double red[32];
    double acc[4] = {0, 0, 0, 0};
    for (int i = threadIdx.x; i < n; i += SH_ONE) {
        double sq = 0.0;
        for (int k = 0; k < d; ++k) {
            const double v = P[(size_t)i * d + k];
            acc[k] += v;
            sq += v * v;
        }
        acc[3] += sq;
    }
    for (int k = 0; k < 4; ++k) {
        const double r = block_sum<SH_ONE>(acc[k], red);
        if (threadIdx.x == 0) {
            if (k < d) out[k] = r;
            if (k == 3) {
                out[d] = r;
                out[d + 1] = (double)n;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// flow start: omega from X and the GLOBAL Y sums (resolve_omega,
// sinkhorn.py:136-148), centrings, warm potentials, control words.  A planner
// that already stopped (plan_state != 0) marks both solves done: the whole
// flow is then a chain of no-ops.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SH_ONE)
    shard_init_kernel(const double* __restrict__ X, int n, int d, const double* __restrict__ ysum,
                      double omega_fixed, double unit, const double* warm_f, const double* warm_p,
                      const int* warm_valid, double* scal_x, double* scal_s, double* f, double* p,
                      int* ctl, unsigned long long* eslot, const int* plan_state) {
    __shared__ double red[32];
    __shared__ double s_sum[4];
    const bool skip = plan_state && *((volatile const int*)plan_state) != 0;
    double acc[4] = {0, 0, 0, 0};
    for (int i = threadIdx.x; i < n; i += SH_ONE) {
        double sq = 0.0;
        for (int k = 0; k < d; ++k) {
            const double v = X[(size_t)i * d + k];
            acc[k] += v;
            sq += v * v;
        }
        acc[3] += sq;
    }
    for (int k = 0; k < 4; ++k) {
        const double r = block_sum<SH_ONE>(acc[k], red);
        if (threadIdx.x == 0) s_sum[k] = r;
    }
    __syncthreads();
    const double m = ysum[d + 1];
    double mx[3] = {0, 0, 0}, my[3] = {0, 0, 0}, dot = 0.0;
    for (int k = 0; k < d; ++k) {
        mx[k] = s_sum[k] / n;
        my[k] = ysum[k] / m;
        dot += mx[k] * my[k];
    }
    const double mx2 = s_sum[3] / n, my2 = ysum[d] / m;
    double w = omega_fixed;
    if (!(w > 0.0)) {
        w = SH_AUTO_OMEGA * (mx2 + my2 - 2.0 * dot);
        if (!(w >= SH_OMEGA_FLOOR)) w = (w != w) ? w : SH_OMEGA_FLOOR;
    }
    if (threadIdx.x == 0) {
        for (int which = 0; which < 2; ++which) {
            double* sc = which ? scal_s : scal_x;
            for (int k = 0; k < 16; ++k) sc[k] = 0.0;
            sc[SC_OMEGA] = w;
            sc[SC_S] = unit / w;
            for (int k = 0; k < d; ++k) {
                sc[SC_C + k] = which ? mx[k] : 0.5 * (mx[k] + my[k]);
                sc[SC_MX + k] = mx[k];
                sc[SC_MY + k] = my[k];
            }
            sc[SC_MX2] = mx2;
            sc[SC_MY2] = my2;
        }
        ctl[CTL_DONE_X] = skip ? 1 : 0;
        ctl[CTL_DONE_P] = skip ? 1 : 0;
        ctl[CTL_IT_X] = 0;
        ctl[CTL_IT_P] = 0;
        ctl[CTL_CNT_X] = 0;
        ctl[CTL_CNT_P] = 0;
        ctl[CTL_CNT_F] = 0;
        ctl[CTL_SKIP] = skip ? 1 : 0;
        eslot[0] = 0ull;
        eslot[1] = 0ull;
    }
    const bool vf = warm_valid && warm_valid[0] != 0;
    const bool vp = warm_valid && warm_valid[1] != 0;
    for (int i = threadIdx.x; i < n; i += SH_ONE) {
        f[i] = vf ? warm_f[i] : 0.0;
        p[i] = vp ? warm_p[i] : 0.0;
    }
}

// Last-block election after a grid-strided pass: returns true in every thread
// of the block that arrived last (all other blocks' global writes visible).
__device__ __forceinline__ bool sh_last_block(int* counter) {
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(counter, 1);
        s_last = (prev == (int)gridDim.x - 1) ? 1 : 0;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

__device__ __forceinline__ double sh_block_max(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, v, o);
        v = (u > v || u != u) ? u : v;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double b = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) b = (red[k] > b || red[k] != red[k]) ? red[k] : b;
    return b;
}

// ---------------------------------------------------------------------------
// cross solve: combine the gathered shard partials of the f-update
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(SH_BLOCK)
    shard_cross_merge_kernel(int n, int R, const double* __restrict__ gath,
                             const double* __restrict__ scal, double loga, double tol,
                             int max_iters, double* f, double* fnext, double* rs, double* mass,
                             double* ybar, int* ctl, unsigned long long* eslot, double* stat) {
    __shared__ double red[32];
    if (*((volatile const int*)(ctl + CTL_DONE_X)) != 0) return;
    const double w = scal[SC_OMEGA];
    const size_t ld = (size_t)n * (D + 1);
    double emax = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double M = -INFINITY;
        for (int r = 0; r < R; ++r) M = fmax(M, gath[r * ld + (size_t)i * (D + 1)]);
        const double Mb = (M > -INFINITY && M < INFINITY) ? M : 0.0;
        double S = 0.0, A[D];
#pragma unroll
        for (int q = 0; q < D; ++q) A[q] = 0.0;
        for (int r = 0; r < R; ++r) {  // fixed rank order
            const double* g = gath + r * ld + (size_t)i * (D + 1);
            const double e = exp(g[0] - Mb);
            S += e;
#pragma unroll
            for (int q = 0; q < D; ++q) A[q] += e * g[1 + q];
        }
        const double L = Mb + log(S);
        const double fi = f[i];
        const double upd = w * (loga - L);
        double delta = (fi - upd) / w;
        if (delta > SH_EXP_CLIP) delta = SH_EXP_CLIP;  // NaN passes
        const double e = fabs(expm1(delta));
        emax = (e > emax || e != e) ? e : emax;
        rs[i] = exp(delta + loga);
        mass[i] = exp(fi / w + L);
#pragma unroll
        for (int q = 0; q < D; ++q) ybar[(size_t)i * D + q] = A[q] / S;
        fnext[i] = upd;
    }
    const double b = sh_block_max(emax, red);
    if (threadIdx.x == 0 && b != 0.0) atomic_max_nonneg(eslot, b);
    if (!sh_last_block(ctl + CTL_CNT_X)) return;
    // decision on the replicated error: identical on every rank
    __shared__ int s_done;
    if (threadIdx.x == 0) {
        const double err = __longlong_as_double((long long)atomicAdd(eslot, 0ull)) / n;
        const int it = ctl[CTL_IT_X] + 1;
        ctl[CTL_IT_X] = it;
        const bool conv = err <= tol;
        s_done = (conv || it >= max_iters) ? 1 : 0;
        if (s_done) {
            stat[0] = err;
            stat[1] = (double)it;
            stat[2] = conv ? 1.0 : 0.0;
            stat[3] = 0.0;
            ctl[CTL_DONE_X] = 1;
        }
        eslot[0] = 0ull;
        ctl[CTL_CNT_X] = 0;
    }
    __syncthreads();
    if (!s_done)  // f <- f_new for the next iteration (f stays pre-update at the stop)
        for (int i = threadIdx.x; i < n; i += blockDim.x) f[i] = fnext[i];
}

// ---------------------------------------------------------------------------
// self term, rows [row0, row0 + nown) of X: per-row update into the send buffer
//   send[li] = {p_new, rho, mass, e, xbar (D)}
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(SH_BLOCK)
    shard_self_rows_kernel(int row0, int nown, const double* __restrict__ Lb,
                           const double* __restrict__ scal, double loga, const double* __restrict__ p,
                           double* __restrict__ send, const int* ctl) {
    if (*((volatile const int*)(ctl + CTL_DONE_P)) != 0) return;
    const double w = scal[SC_OMEGA];
    for (int li = blockIdx.x * blockDim.x + threadIdx.x; li < nown; li += gridDim.x * blockDim.x) {
        const double* lb = Lb + (size_t)li * (D + 1);
        const double L = lb[0];
        const double pi = p[row0 + li];
        const double target = w * (loga - L);
        double delta = (pi - target) / w;
        if (delta > SH_EXP_CLIP) delta = SH_EXP_CLIP;
        double* o = send + (size_t)li * (D + 4);
        o[0] = 0.5 * (pi + target);
        o[1] = exp(delta + loga);
        o[2] = exp(pi / w + L);
        o[3] = fabs(expm1(delta));
#pragma unroll
        for (int q = 0; q < D; ++q) o[4 + q] = lb[1 + q];
    }
}

__device__ __forceinline__ int shard_of_row(int i, int n, int R) {
    // balanced contiguous shards: rank r owns [n r / R, n (r+1) / R)
    int r = (int)(((long long)i * R) / n);
    while (r + 1 < R && (long long)n * (r + 1) / R <= i) ++r;
    while (r > 0 && (long long)n * r / R > i) --r;
    return r;
}

template <int D>
__global__ void __launch_bounds__(SH_BLOCK)
    shard_self_commit_kernel(int n, int R, int chunk, const double* __restrict__ gath, double tol,
                             int max_iters, double* p, double* pnext, double* rho, double* massp,
                             double* xbar, int* ctl, unsigned long long* eslot, double* stat) {
    __shared__ double red[32];
    if (*((volatile const int*)(ctl + CTL_DONE_P)) != 0) return;
    double emax = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = shard_of_row(i, n, R);
        const int li = i - (int)((long long)n * r / R);
        const double* o = gath + ((size_t)r * chunk + li) * (D + 4);
        pnext[i] = o[0];
        rho[i] = o[1];
        massp[i] = o[2];
        const double e = o[3];
        emax = (e > emax || e != e) ? e : emax;
#pragma unroll
        for (int q = 0; q < D; ++q) xbar[(size_t)i * D + q] = o[4 + q];
    }
    const double b = sh_block_max(emax, red);
    if (threadIdx.x == 0 && b != 0.0) atomic_max_nonneg(eslot + 1, b);
    if (!sh_last_block(ctl + CTL_CNT_P)) return;
    __shared__ int s_done;
    if (threadIdx.x == 0) {
        const double err = __longlong_as_double((long long)atomicAdd(eslot + 1, 0ull)) / n;
        const int it = ctl[CTL_IT_P] + 1;
        ctl[CTL_IT_P] = it;
        const bool conv = err <= tol;
        s_done = (conv || it >= max_iters) ? 1 : 0;
        if (s_done) {
            stat[0] = err;
            stat[1] = (double)it;
            stat[2] = conv ? 1.0 : 0.0;
            stat[3] = 0.0;
            ctl[CTL_DONE_P] = 1;
        }
        eslot[1] = 0ull;
        ctl[CTL_CNT_P] = 0;
    }
    __syncthreads();
    if (!s_done)
        for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = pnext[i];
}

// ---------------------------------------------------------------------------
// envelope gradient (sinkhorn.py:383-391), FlowError test (:370-373), warm
// state (:393-395), planner hooks (flow_log row, convergence, plan_state)
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(SH_BLOCK)
    shard_flow_finish_kernel(const double* __restrict__ X, int n, const double* rs,
                             const double* mass, const double* ybar, const double* rho,
                             const double* massp, const double* xbar, const double* stat_x,
                             const double* stat_p, double tol, const double* f, const double* p,
                             double* warm_f, double* warm_p, int* warm_valid, double* flow,
                             double* fstat, const double* scal, int* plan_state, int iteration,
                             double* flow_log, double conv_tol, double* part, int* ctl) {
    __shared__ double red[32];
    if (*((volatile const int*)(ctl + CTL_SKIP)) != 0) return;
    const double ex = stat_x[0], ep = stat_p[0];
    const double worst = (ex > ep || ex != ex) ? ex : ep;
    const bool flow_error = worst > 100.0 * tol;
    double norm_acc = 0.0;
    if (!flow_error) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            double sq = 0.0;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                const double x = X[(size_t)i * D + q];
                const double grad = 2.0 * (rs[i] * x - mass[i] * ybar[(size_t)i * D + q]) -
                                    2.0 * (rho[i] * x - massp[i] * xbar[(size_t)i * D + q]);
                flow[(size_t)i * D + q] = -grad;
                sq += grad * grad;
            }
            norm_acc += sqrt(sq);
            if (warm_f) {
                warm_f[i] = f[i];
                warm_p[i] = p[i];
            }
        }
    }
    const double blk = block_sum<SH_BLOCK>(norm_acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = blk;
    if (!sh_last_block(ctl + CTL_CNT_F)) return;
    if (threadIdx.x != 0) return;
    double total = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) total += part[b];  // fixed order
    ctl[CTL_CNT_F] = 0;
    const double mean_mag = total / n;
    fstat[0] = worst;
    fstat[1] = (stat_x[2] != 0.0 && stat_p[2] != 0.0) ? 1.0 : 0.0;
    fstat[2] = flow_error ? 1.0 : 0.0;
    fstat[3] = flow_error ? NAN : mean_mag;
    fstat[4] = scal[SC_OMEGA];
    fstat[5] = stat_x[1];
    fstat[6] = stat_p[1];
    fstat[7] = 0.0;
    if (!flow_error && warm_valid) {
        warm_valid[0] = 1;
        warm_valid[1] = 1;
    }
    if (plan_state) {
        if (flow_error) {
            plan_state[FCB_STATE_STOP] = 2;
            plan_state[FCB_STATE_STAGE] = 2;
            plan_state[FCB_STATE_ITER] = iteration;
            plan_state[FCB_STATE_INDEX] = -1;
        } else {
            double* lg = flow_log + 4 * (size_t)iteration;
            lg[0] = mean_mag;
            lg[1] = fstat[5];
            lg[2] = fstat[6];
            lg[3] = worst;
            plan_state[FCB_STATE_FLOWS] = iteration + 1;
            if (mean_mag < conv_tol) plan_state[FCB_STATE_STOP] = 1;
        }
    }
}

// ---------------------------------------------------------------------------
// SVGD with sharded sources
// ---------------------------------------------------------------------------
int stein_partial(int precision, const double* X, int n, int d, int col0, int ncols,
                  const double* scores, const double* hstat, double* part, const int* gate,
                  void* ws, size_t ws_bytes, cudaStream_t st);
size_t stein_partial_ws_bytes(int precision, int n, int nc, int d);
size_t median_ws_bytes(int n);
long long median_tiles(int n);
size_t median_hist_offset();
int median_shard_init(int n, void* ws, size_t ws_bytes, const int* gate, cudaStream_t st);
int median_shard_pass(const double* X, int n, int d, int pass, long long t_lo, long long t_hi,
                      void* ws, const int* gate, cudaStream_t st);
int median_shard_select(int n, int pass, void* ws, const int* gate, cudaStream_t st);
int median_shard_finish(int n, double log_np1, double* hstat, void* ws, const int* gate,
                        cudaStream_t st);

template <int D>
__global__ void __launch_bounds__(SH_BLOCK)
    stein_combine_kernel(int n, int R, const double* __restrict__ parts,
                         const double* __restrict__ X, const double* __restrict__ hstat,
                         double* __restrict__ flow, double* part_norm, int* counter,
                         double* fstat, int* plan_state, int iteration, double* flow_log,
                         double conv_tol) {
    __shared__ double red[32];
    if (plan_state && *((volatile const int*)plan_state) != 0) return;
    const double h = hstat[0];
    const double two_over_h = 2.0 / h, inv_n = 1.0 / n;
    const size_t ld = (size_t)n * (D + 1);
    double norm_acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double K = 0.0, A[D];
#pragma unroll
        for (int q = 0; q < D; ++q) A[q] = 0.0;
        for (int r = 0; r < R; ++r) {  // fixed rank order
            const double* pp = parts + r * ld + (size_t)i * (D + 1);
            K += pp[0];
#pragma unroll
            for (int q = 0; q < D; ++q) A[q] += pp[1 + q];
        }
        double sq = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) {
            // partial sums are centred on X[0] (fcb_stein_partial)
            const double xc = X[(size_t)i * D + q] - X[q];
            const double v = inv_n * (A[q] + two_over_h * xc * K);
            flow[(size_t)i * D + q] = v;
            sq += v * v;
        }
        norm_acc += sqrt(sq);
    }
    const double blk = block_sum<SH_BLOCK>(norm_acc, red);
    if (threadIdx.x == 0) part_norm[blockIdx.x] = blk;
    if (!sh_last_block(counter)) return;
    if (threadIdx.x != 0) return;
    double total = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) total += part_norm[b];
    *counter = 0;
    const double mean_mag = total / n;
    if (fstat) {
        fstat[0] = 0.0;
        fstat[1] = 1.0;
        fstat[2] = 0.0;
        fstat[3] = mean_mag;
        fstat[4] = hstat[0];
        fstat[5] = hstat[2];
        fstat[6] = hstat[1];
        fstat[7] = 0.0;
    }
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

}  // namespace fcb

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using namespace fcb;

#define CS(s) static_cast<cudaStream_t>(s)

#define SH_DISPATCH(d, CALL)                  \
    switch (d) {                              \
        case 1: { constexpr int DD = 1; CALL; } break; \
        case 2: { constexpr int DD = 2; CALL; } break; \
        case 3: { constexpr int DD = 3; CALL; } break; \
        default: return fail(FCB_ENOTSUP, "point dimension must be 1, 2 or 3"); \
    }

extern "C" {

FCB_API int fcb_point_sums(const double* P, int n, int d, double* out, fcb_stream_t stream) {
    if (n < 1 || d < 1 || d > 3) return fail(FCB_EINPUT, "point_sums: bad shape");
    point_sums_kernel<<<1, SH_ONE, 0, CS(stream)>>>(P, n, d, out);
    FCB_LAUNCHED("point_sums_kernel");
    return FCB_OK;
}

FCB_API size_t fcb_lse_sweep_workspace_bytes(int precision, int nr, int ns, int d) {
    return ot_ws_bytes(FCB_OT_SWEEP, precision, nr, ns, d);
}

FCB_API int fcb_lse_sweep(int precision, const double* R, int nr, const double* S, int ns, int d,
                          const double* scal, const double* pot, const double* row_est,
                          double row_logw, double out_scale, double out_shift, double* out,
                          double* bary, const int* gate, void* ws, size_t ws_bytes,
                          fcb_stream_t stream) {
    return lse_sweep(precision, R, nr, S, ns, d, scal, pot, row_est, row_logw, out_scale,
                     out_shift, out, bary, gate, ws, ws_bytes, CS(stream));
}

FCB_API int fcb_shard_init(int precision, const double* X, int n, int d, const double* ysum,
                           double omega_fixed, const double* warm_f, const double* warm_p,
                           const int* warm_valid, double* scal_x, double* scal_s, double* f,
                           double* p, int* ctl, unsigned long long* eslot, const int* plan_state,
                           fcb_stream_t stream) {
    if (n < 1 || d < 1 || d > 3) return fail(FCB_EINPUT, "shard_init: bad shape");
    const double unit = precision == FCB_FP64 ? 1.0 : kLog2e;
    shard_init_kernel<<<1, SH_ONE, 0, CS(stream)>>>(X, n, d, ysum, omega_fixed, unit, warm_f,
                                                    warm_p, warm_valid, scal_x, scal_s, f, p, ctl,
                                                    eslot, plan_state);
    FCB_LAUNCHED("shard_init_kernel");
    return FCB_OK;
}

FCB_API int fcb_shard_cross_merge(int n, int d, int R, const double* gathered, const double* scal,
                                  double tol, int max_iters, double* f, double* fnext, double* rs,
                                  double* mass, double* ybar, int* ctl, unsigned long long* eslot,
                                  double* stat, fcb_stream_t stream) {
    const double loga = -log((double)n);
    SH_DISPATCH(d, (shard_cross_merge_kernel<DD><<<sh_blocks(n), SH_BLOCK, 0, CS(stream)>>>(
                       n, R, gathered, scal, loga, tol, max_iters, f, fnext, rs, mass, ybar, ctl,
                       eslot, stat)));
    FCB_LAUNCHED("shard_cross_merge_kernel");
    return FCB_OK;
}

FCB_API int fcb_shard_self_rows(int n, int d, int row0, int nown, const double* Lb,
                                const double* scal, const double* p, double* send, const int* ctl,
                                fcb_stream_t stream) {
    const double loga = -log((double)n);
    SH_DISPATCH(d, (shard_self_rows_kernel<DD><<<sh_blocks(nown), SH_BLOCK, 0, CS(stream)>>>(
                       row0, nown, Lb, scal, loga, p, send, ctl)));
    FCB_LAUNCHED("shard_self_rows_kernel");
    return FCB_OK;
}

FCB_API int fcb_shard_self_commit(int n, int d, int R, int chunk, const double* gathered,
                                  double tol, int max_iters, double* p, double* pnext, double* rho,
                                  double* massp, double* xbar, int* ctl, unsigned long long* eslot,
                                  double* stat, fcb_stream_t stream) {
    SH_DISPATCH(d, (shard_self_commit_kernel<DD><<<sh_blocks(n), SH_BLOCK, 0, CS(stream)>>>(
                       n, R, chunk, gathered, tol, max_iters, p, pnext, rho, massp, xbar, ctl,
                       eslot, stat)));
    FCB_LAUNCHED("shard_self_commit_kernel");
    return FCB_OK;
}

FCB_API size_t fcb_shard_finish_workspace_bytes(int n) {
    return (size_t)sh_blocks(n) * sizeof(double) + 256;
}

FCB_API int fcb_shard_flow_finish(const double* X, int n, int d, const double* rs,
                                  const double* mass, const double* ybar, const double* rho,
                                  const double* massp, const double* xbar, const double* stat_x,
                                  const double* stat_p, double tol, const double* f,
                                  const double* p, double* warm_f, double* warm_p, int* warm_valid,
                                  double* flow, double* fstat, const double* scal, int* plan_state,
                                  int iteration, double* flow_log, double conv_tol, int* ctl,
                                  void* ws, size_t ws_bytes, fcb_stream_t stream) {
    if (ws_bytes < fcb_shard_finish_workspace_bytes(n))
        return fail(FCB_EWORKSPACE, "shard_flow_finish workspace too small");
    SH_DISPATCH(d, (shard_flow_finish_kernel<DD><<<sh_blocks(n), SH_BLOCK, 0, CS(stream)>>>(
                       X, n, rs, mass, ybar, rho, massp, xbar, stat_x, stat_p, tol, f, p, warm_f,
                       warm_p, warm_valid, flow, fstat, scal, plan_state, iteration, flow_log,
                       conv_tol, static_cast<double*>(ws), ctl)));
    FCB_LAUNCHED("shard_flow_finish_kernel");
    return FCB_OK;
}

FCB_API int fcb_stein_combine(const double* X, int n, int d, int R, const double* parts,
                              const double* hstat, double* flow, double* fstat, int* plan_state,
                              int iteration, double* flow_log, double conv_tol, void* ws,
                              size_t ws_bytes, fcb_stream_t stream) {
    const int blocks = sh_blocks(n);
    if (ws_bytes < (size_t)blocks * sizeof(double) + 64)
        return fail(FCB_EWORKSPACE, "stein_combine workspace too small");
    double* part_norm = static_cast<double*>(ws);
    int* counter = reinterpret_cast<int*>(part_norm + blocks);
    FCB_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), CS(stream)));
    SH_DISPATCH(d, (stein_combine_kernel<DD><<<blocks, SH_BLOCK, 0, CS(stream)>>>(
                       n, R, parts, X, hstat, flow, part_norm, counter, fstat, plan_state,
                       iteration, flow_log, conv_tol)));
    FCB_LAUNCHED("stein_combine_kernel");
    return FCB_OK;
}

FCB_API size_t fcb_stein_combine_workspace_bytes(int n) {
    return (size_t)sh_blocks(n) * sizeof(double) + 64;
}

FCB_API size_t fcb_stein_partial_workspace_bytes(int precision, int n, int nc, int d) {
    return stein_partial_ws_bytes(precision, n, nc, d);
}

FCB_API int fcb_stein_partial(int precision, const double* X, int n, int d, int col0, int ncols,
                              const double* scores, const double* hstat, double* part,
                              const int* gate, void* ws, size_t ws_bytes, fcb_stream_t stream) {
    return stein_partial(precision, X, n, d, col0, ncols, scores, hstat, part, gate, ws, ws_bytes,
                         CS(stream));
}

FCB_API long long fcb_median_tiles(int n) { return median_tiles(n); }
FCB_API size_t fcb_median_hist_offset(void) { return median_hist_offset(); }

FCB_API int fcb_median_shard_init(int n, void* ws, size_t ws_bytes, const int* gate,
                                  fcb_stream_t stream) {
    return median_shard_init(n, ws, ws_bytes, gate, CS(stream));
}

FCB_API int fcb_median_shard_pass(const double* X, int n, int d, int pass, long long tile_lo,
                                  long long tile_hi, void* ws, const int* gate,
                                  fcb_stream_t stream) {
    return median_shard_pass(X, n, d, pass, tile_lo, tile_hi, ws, gate, CS(stream));
}

FCB_API int fcb_median_shard_select(int n, int pass, void* ws, const int* gate,
                                    fcb_stream_t stream) {
    return median_shard_select(n, pass, ws, gate, CS(stream));
}

FCB_API int fcb_median_shard_finish(int n, double log_np1, double* hstat, void* ws,
                                    const int* gate, fcb_stream_t stream) {
    return median_shard_finish(n, log_np1, hstat, ws, gate, CS(stream));
}

}  // extern "C"
