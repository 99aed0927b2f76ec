// dynamics.cu -- RK4 rollout, Jacobians and the flow-matching LQR on device.
//
// Replaces dynamics.py:72-181 (models), :276-312 (rollout), :315-329
// (linearize_along) and lqr.py:154-200 (solve_flow_lqr) plus the control
// update of optimizer.py:259-268.  All arithmetic is float64.  Vector-field
// and RK4 arithmetic use explicitly rounded intrinsics (no FMA contraction)
// in the reference's operation order, so rollouts of the polynomial models
// (single/double integrator, LTI) are bit-identical to numpy's.
//
// The Riccati sweep and the rollout are sequential in time; each problem is
// one thread with its matrices in registers (n <= 6, m <= 3).
#include "fcb_internal.cuh"
#include "lqr_scan.cuh"
#include "plan_scan.cuh"

#include <algorithm>
#include <atomic>

namespace fcb {

#define DADD __dadd_rn
#define DSUB __dsub_rn
#define DMUL __dmul_rn

// ---------------------------------------------------------------------------
// models
// ---------------------------------------------------------------------------
template <int MODEL> struct Model;

template <> struct Model<FCB_MODEL_SINGLE_INTEGRATOR_2D> {
    static constexpr int N = 2, M = 2;
    static constexpr bool LINEAR = true;
    static constexpr bool TRIANGULAR = false;
    __device__ static void f(const double* s, const double* u, const double*, double* out) {
        out[0] = u[0];
        out[1] = u[1];
    }
    __device__ static void jac(const double*, const double*, const double*, double* A, double* B) {
        A[0] = A[1] = A[2] = A[3] = 0.0;
        B[0] = 1.0; B[1] = 0.0; B[2] = 0.0; B[3] = 1.0;
    }
};

template <> struct Model<FCB_MODEL_DIFF_DRIVE> {
    static constexpr int N = 3, M = 2;
    static constexpr bool LINEAR = false;
    // triangular structure: q = (theta) integrates u1; the position
    // derivative depends on (q, u) only -> parallel RK4 rollout
    static constexpr bool TRIANGULAR = true;
    static constexpr int NQ = 1, NP = 2, QOFF = 2;
    __device__ static void qdot(const double* u, double* qd) { qd[0] = u[1]; }
    __device__ static void pdot(const double* q, const double* u, double* pd) {
        pd[0] = DMUL(u[0], cos(q[0]));
        pd[1] = DMUL(u[0], sin(q[0]));
    }
    __device__ static void f(const double* s, const double* u, const double*, double* out) {
        out[0] = DMUL(u[0], cos(s[2]));
        out[1] = DMUL(u[0], sin(s[2]));
        out[2] = u[1];
    }
    __device__ static void jac(const double* s, const double* u, const double*, double* A,
                               double* B) {
        const double st = sin(s[2]), ct = cos(s[2]);
        for (int k = 0; k < 9; ++k) A[k] = 0.0;
        A[0 * 3 + 2] = -DMUL(u[0], st);
        A[1 * 3 + 2] = DMUL(u[0], ct);
        B[0] = ct; B[1] = 0.0;
        B[2] = st; B[3] = 0.0;
        B[4] = 0.0; B[5] = 1.0;
    }
};

template <> struct Model<FCB_MODEL_AIRCRAFT_3D> {
    static constexpr int N = 6, M = 3;
    static constexpr bool LINEAR = false;
    // q = (psi, gamma, v) integrates u; positions depend on q only
    static constexpr bool TRIANGULAR = true;
    static constexpr int NQ = 3, NP = 3, QOFF = 3;
    __device__ static void qdot(const double* u, double* qd) {
        qd[0] = u[0];
        qd[1] = u[1];
        qd[2] = u[2];
    }
    __device__ static void pdot(const double* q, const double*, double* pd) {
        const double vcg = DMUL(q[2], cos(q[1]));
        pd[0] = DMUL(vcg, cos(q[0]));
        pd[1] = DMUL(vcg, sin(q[0]));
        pd[2] = DMUL(q[2], sin(q[1]));
    }
    __device__ static void f(const double* s, const double* u, const double*, double* out) {
        const double psi = s[3], gamma = s[4], v = s[5];
        const double cg = cos(gamma);
        const double vcg = DMUL(v, cg);
        out[0] = DMUL(vcg, cos(psi));
        out[1] = DMUL(vcg, sin(psi));
        out[2] = DMUL(v, sin(gamma));
        out[3] = u[0];
        out[4] = u[1];
        out[5] = u[2];
    }
    __device__ static void jac(const double* s, const double*, const double*, double* A,
                               double* B) {
        const double psi = s[3], gamma = s[4], v = s[5];
        const double sp = sin(psi), cp = cos(psi), sg = sin(gamma), cg = cos(gamma);
        for (int k = 0; k < 36; ++k) A[k] = 0.0;
        A[0 * 6 + 3] = -DMUL(DMUL(v, cg), sp);
        A[0 * 6 + 4] = -DMUL(DMUL(v, sg), cp);
        A[0 * 6 + 5] = DMUL(cg, cp);
        A[1 * 6 + 3] = DMUL(DMUL(v, cg), cp);
        A[1 * 6 + 4] = -DMUL(DMUL(v, sg), sp);
        A[1 * 6 + 5] = DMUL(cg, sp);
        A[2 * 6 + 4] = DMUL(v, cg);
        A[2 * 6 + 5] = sg;
        for (int k = 0; k < 18; ++k) B[k] = 0.0;
        B[3 * 3 + 0] = 1.0;
        B[4 * 3 + 1] = 1.0;
        B[5 * 3 + 2] = 1.0;
    }
};

template <> struct Model<FCB_MODEL_DOUBLE_INTEGRATOR_2D> {
    static constexpr int N = 4, M = 2;
    static constexpr bool LINEAR = true;
    static constexpr bool TRIANGULAR = false;
    __device__ static void f(const double* s, const double* u, const double*, double* out) {
        out[0] = s[2];
        out[1] = s[3];
        out[2] = u[0];
        out[3] = u[1];
    }
    __device__ static void jac(const double*, const double*, const double*, double* A, double* B) {
        for (int k = 0; k < 16; ++k) A[k] = 0.0;
        A[0 * 4 + 2] = 1.0;
        A[1 * 4 + 3] = 1.0;
        for (int k = 0; k < 8; ++k) B[k] = 0.0;
        B[2 * 2 + 0] = 1.0;
        B[3 * 2 + 1] = 1.0;
    }
};

// LTI: f = A s + B u with A, B in model params (row-major); evaluated as the
// matrix-vector products numpy would form (left-to-right dot products).
template <int N_, int M_> struct Lti {
    static constexpr int N = N_, M = M_;
    static constexpr bool LINEAR = true;
    static constexpr bool TRIANGULAR = false;
    __device__ static void f(const double* s, const double* u, const double* prm, double* out) {
        const double* A = prm;
        const double* B = prm + N * N;
        for (int r = 0; r < N; ++r) {
            double a = 0.0;
            for (int k = 0; k < N; ++k) a = DADD(a, DMUL(A[r * N + k], s[k]));
            double b = 0.0;
            for (int k = 0; k < M; ++k) b = DADD(b, DMUL(B[r * M + k], u[k]));
            out[r] = DADD(a, b);
        }
    }
    __device__ static void jac(const double*, const double*, const double* prm, double* A,
                               double* B) {
        for (int k = 0; k < N * N; ++k) A[k] = prm[k];
        for (int k = 0; k < N * M; ++k) B[k] = prm[N * N + k];
    }
};

// ---------------------------------------------------------------------------
// rollout
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool all_finite(const double* v, int n) {
    bool ok = true;
    for (int k = 0; k < n; ++k) ok = ok && isfinite(v[k]);
    return ok;
}

constexpr int RO_CHUNK = 256;

// One warp per rollout: all lanes stage a chunk of controls into shared
// memory (coalesced), lane 0 integrates the chunk, then all lanes write the
// states and workspace points back.  The sequential RK4 chain never waits on
// a global load.
template <class Mdl>
__global__ void __launch_bounds__(32) rollout_kernel(const double* __restrict__ prm,
                                                    const double* __restrict__ s0,
                                                    const double* __restrict__ U, int T, double dt,
                                                    double* __restrict__ S, int d,
                                                    const double* __restrict__ P,
                                                    double* __restrict__ X, int* status,
                                                    int* plan_state, int iteration) {
    constexpr int N = Mdl::N, M = Mdl::M;
    __shared__ double sU[RO_CHUNK * M];
    __shared__ double sS[RO_CHUNK * N];
    __shared__ double sP[3 * N];
    __shared__ int s_fail;
    const int lane = threadIdx.x;
    if (plan_state && *((volatile int*)plan_state) != 0) return;
    for (int i = lane; i < d * N; i += 32) sP[i] = P ? P[i] : 0.0;
    if (lane == 0) s_fail = -1;
    double s[N];
    for (int j = 0; j < N; ++j) s[j] = s0[j];
    if (lane < N) S[lane] = s0[lane];
    const double half = DMUL(0.5, dt);
    const double sixth = dt / 6.0;
    for (int c0 = 0; c0 < T; c0 += RO_CHUNK) {
        const int len = min(RO_CHUNK, T - c0);
        for (int i = lane; i < len * M; i += 32) sU[i] = U[(size_t)c0 * M + i];
        __syncwarp();
        if (lane == 0 && s_fail < 0) {
            double u[M], k1[N], k2[N], k3[N], k4[N], tmp[N];
            for (int k = 0; k < len; ++k) {
                for (int j = 0; j < M; ++j) u[j] = sU[k * M + j];
                Mdl::f(s, u, prm, k1);
                for (int j = 0; j < N; ++j) tmp[j] = DADD(s[j], DMUL(half, k1[j]));
                Mdl::f(tmp, u, prm, k2);
                for (int j = 0; j < N; ++j) tmp[j] = DADD(s[j], DMUL(half, k2[j]));
                Mdl::f(tmp, u, prm, k3);
                for (int j = 0; j < N; ++j) tmp[j] = DADD(s[j], DMUL(dt, k3[j]));
                Mdl::f(tmp, u, prm, k4);
                for (int j = 0; j < N; ++j) {
                    const double inner = DADD(DADD(k1[j], DMUL(2.0, DADD(k2[j], k3[j]))), k4[j]);
                    s[j] = DADD(s[j], DMUL(sixth, inner));
                }
                if (!all_finite(s, N)) {
                    s_fail = c0 + k + 1;
                    break;
                }
                for (int j = 0; j < N; ++j) sS[k * N + j] = s[j];
            }
        }
        __syncwarp();
        const int fail = s_fail;
        const int valid = (fail < 0) ? len : (fail - 1 - c0);
        for (int i = lane; i < valid * N; i += 32) S[(size_t)(c0 + 1) * N + i] = sS[i];
        if (X)
            for (int i = lane; i < valid * d; i += 32) {
                const int k = i / d, r = i % d;
                double a = 0.0;
                for (int j = 0; j < N; ++j) a = DADD(a, DMUL(sS[k * N + j], sP[r * N + j]));
                X[(size_t)(c0 + k) * d + r] = a;
            }
        __syncwarp();
        if (fail >= 0) break;
    }
    if (lane == 0) {
        if (status) *status = s_fail;
        if (plan_state && s_fail >= 0) {
            plan_state[FCB_STATE_STOP] = 2;
            plan_state[FCB_STATE_STAGE] = 1;
            plan_state[FCB_STATE_ITER] = iteration;
            plan_state[FCB_STATE_INDEX] = s_fail;
        }
    }
}

template <class Mdl>
__global__ void linearize_kernel(const double* __restrict__ prm, const double* __restrict__ S,
                                 const double* __restrict__ U, int T, double* __restrict__ A,
                                 double* __restrict__ B) {
    constexpr int N = Mdl::N, M = Mdl::M;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < T; k += gridDim.x * blockDim.x) {
        double s[N], u[M], a[N * N], b[N * M];
        for (int j = 0; j < N; ++j) s[j] = S[(size_t)k * N + j];
        for (int j = 0; j < M; ++j) u[j] = U[(size_t)k * M + j];
        Mdl::jac(s, u, prm, a, b);
        for (int j = 0; j < N * N; ++j) A[(size_t)k * N * N + j] = a[j];
        for (int j = 0; j < N * M; ++j) B[(size_t)k * N * M + j] = b[j];
    }
}

// ---------------------------------------------------------------------------
// flow-matching LQR (lqr.py:154-200)
// ---------------------------------------------------------------------------
// Source of per-step Jacobians: explicit arrays or a model evaluated along
// (S, U) on the fly.
template <int N, int M>
struct ArrayJac {
    const double* A;
    const double* B;
    __device__ void get(int k, double* a, double* b) const {
        for (int j = 0; j < N * N; ++j) a[j] = A[(size_t)k * N * N + j];
        for (int j = 0; j < N * M; ++j) b[j] = B[(size_t)k * N * M + j];
    }
};

template <class Mdl>
struct ModelJac {
    const double* prm;
    const double* S;
    const double* U;
    __device__ void get(int k, double* a, double* b) const {
        double s[Mdl::N], u[Mdl::M];
        for (int j = 0; j < Mdl::N; ++j) s[j] = S[(size_t)k * Mdl::N + j];
        for (int j = 0; j < Mdl::M; ++j) u[j] = U[(size_t)k * Mdl::M + j];
        Mdl::jac(s, u, prm, a, b);
    }
};

// Source of the state-space flow a[k]: explicit (T, n) or a workspace flow
// (T, d) lifted by the projection matrix (lift_flow, lqr.py:140-142).
template <int N>
struct ArrayFlow {
    const double* a;
    __device__ void get(int k, double* out) const {
        for (int j = 0; j < N; ++j) out[j] = a[(size_t)k * N + j];
    }
};
template <int N>
struct LiftedFlow {
    const double* w;
    const double* P;
    int d;
    __device__ void get(int k, double* out) const {
        for (int j = 0; j < N; ++j) {
            double v = 0.0;
            for (int r = 0; r < d; ++r) v = DADD(v, DMUL(w[(size_t)k * d + r], P[r * N + j]));
            out[j] = v;
        }
    }
};

// The Riccati phase (lqr_split.cuh) as three launches over the whole GPU:
// warp chunk aggregates + in-CTA suffix scan, the suffix scan over CTAs, and
// the per-step re-walk emitting the gains.  The plan_* variants evaluate the
// model's Jacobians along (S, U) on the fly and are gated by the planner
// status word.
template <int N, int M>
__global__ void __launch_bounds__(RW_BLOCK) ric_arrays_k1(RicArgs p, const double* A,
                                                          const double* B) {
    ArrayJac<N, M> jac{A, B};
    riccati_k1<N, M>(jac, p);
}
template <int N, int M>
__global__ void __launch_bounds__(RW_BLOCK) ric_arrays_k3(RicArgs p, const double* A,
                                                          const double* B) {
    ArrayJac<N, M> jac{A, B};
    riccati_k3<N, M>(jac, p);
}

__device__ __forceinline__ bool ric_gated(const RicArgs& p) {
    return p.plan_state && *((volatile const int*)p.plan_state) != 0;
}

template <class Mdl>
__global__ void __launch_bounds__(RW_BLOCK) plan_ric_k1(RicArgs p, const double* prm,
                                                        const double* S, const double* U) {
    if (ric_gated(p)) return;
    ModelJac<Mdl> jac{prm, S, U};
    riccati_k1<Mdl::N, Mdl::M>(jac, p);
}
template <class Mdl>
__global__ void __launch_bounds__(RW_BLOCK) plan_ric_k3(RicArgs p, const double* prm,
                                                        const double* S, const double* U) {
    if (ric_gated(p)) return;
    ModelJac<Mdl> jac{prm, S, U};
    riccati_k3<Mdl::N, Mdl::M>(jac, p);
}

template <int N, int M>
__global__ void __launch_bounds__(32 * RW_K2_WARPS) ric_k2(RicArgs p) {
    if (ric_gated(p)) return;
    riccati_k2<N, M>(p);
}

__global__ void ric_finish_kernel(RicArgs p) {
    if (ric_gated(p)) return;
    riccati_finish(p);
}

// Launch one Riccati kernel with its dynamic shared memory (opt-in > 48 KB).
template <typename... Args>
static void ric_launch(void (*kern)(Args...), int grid, int warps, size_t smem, cudaStream_t st,
                       Args... args) {
    cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 32 * warps, smem, st>>>(args...);
}

// Riccati phase on explicit or model Jacobians: K1, K2, K3 (+ finish).
template <int N, int M, class K1, class K3, typename... J>
static int ric_phase(K1 k1, K3 k3, const RicArgs& r, cudaStream_t st, bool finish, J... jargs) {
    ric_launch(k1, r.nblk, RW_WARPS, rw_smem_bytes<N, M>(RW_WARPS), st, r, jargs...);
    ric_launch(ric_k2<N, M>, 1, RW_K2_WARPS, rw_smem_bytes<N, M>(RW_K2_WARPS), st, r);
    ric_launch(k3, r.nblk, RW_WARPS, rw_smem_bytes<N, M>(RW_WARPS), st, r, jargs...);
    if (finish) ric_finish_kernel<<<1, 32, 0, st>>>(r);
    return finish ? 4 : 3;
}

static int ric_max_blocks() { return sm_count(); }

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
#define FCB_LTI_DISPATCH(KERNEL_LAUNCH)                                                      \
    switch (ns * 4 + m) {                                                                    \
        case 1 * 4 + 1: { using Mdl = Lti<1, 1>; KERNEL_LAUNCH; } break;                     \
        case 1 * 4 + 2: { using Mdl = Lti<1, 2>; KERNEL_LAUNCH; } break;                     \
        case 1 * 4 + 3: { using Mdl = Lti<1, 3>; KERNEL_LAUNCH; } break;                     \
        case 2 * 4 + 1: { using Mdl = Lti<2, 1>; KERNEL_LAUNCH; } break;                     \
        case 2 * 4 + 2: { using Mdl = Lti<2, 2>; KERNEL_LAUNCH; } break;                     \
        case 2 * 4 + 3: { using Mdl = Lti<2, 3>; KERNEL_LAUNCH; } break;                     \
        case 3 * 4 + 1: { using Mdl = Lti<3, 1>; KERNEL_LAUNCH; } break;                     \
        case 3 * 4 + 2: { using Mdl = Lti<3, 2>; KERNEL_LAUNCH; } break;                     \
        case 3 * 4 + 3: { using Mdl = Lti<3, 3>; KERNEL_LAUNCH; } break;                     \
        case 4 * 4 + 1: { using Mdl = Lti<4, 1>; KERNEL_LAUNCH; } break;                     \
        case 4 * 4 + 2: { using Mdl = Lti<4, 2>; KERNEL_LAUNCH; } break;                     \
        case 4 * 4 + 3: { using Mdl = Lti<4, 3>; KERNEL_LAUNCH; } break;                     \
        case 5 * 4 + 1: { using Mdl = Lti<5, 1>; KERNEL_LAUNCH; } break;                     \
        case 5 * 4 + 2: { using Mdl = Lti<5, 2>; KERNEL_LAUNCH; } break;                     \
        case 5 * 4 + 3: { using Mdl = Lti<5, 3>; KERNEL_LAUNCH; } break;                     \
        case 6 * 4 + 1: { using Mdl = Lti<6, 1>; KERNEL_LAUNCH; } break;                     \
        case 6 * 4 + 2: { using Mdl = Lti<6, 2>; KERNEL_LAUNCH; } break;                     \
        case 6 * 4 + 3: { using Mdl = Lti<6, 3>; KERNEL_LAUNCH; } break;                     \
        default: return fail(FCB_ENOTSUP, "LTI model needs 1<=ns<=6 and 1<=m<=3");           \
    }

#define FCB_MODEL_DISPATCH(KERNEL_LAUNCH)                                                    \
    switch (model) {                                                                         \
        case FCB_MODEL_SINGLE_INTEGRATOR_2D: {                                               \
            using Mdl = Model<FCB_MODEL_SINGLE_INTEGRATOR_2D>; KERNEL_LAUNCH; } break;       \
        case FCB_MODEL_DIFF_DRIVE: {                                                         \
            using Mdl = Model<FCB_MODEL_DIFF_DRIVE>; KERNEL_LAUNCH; } break;                 \
        case FCB_MODEL_AIRCRAFT_3D: {                                                        \
            using Mdl = Model<FCB_MODEL_AIRCRAFT_3D>; KERNEL_LAUNCH; } break;                \
        case FCB_MODEL_DOUBLE_INTEGRATOR_2D: {                                               \
            using Mdl = Model<FCB_MODEL_DOUBLE_INTEGRATOR_2D>; KERNEL_LAUNCH; } break;       \
        case FCB_MODEL_LTI: FCB_LTI_DISPATCH(KERNEL_LAUNCH) break;                           \
        default: return fail(FCB_ENOTSUP, "unknown device model id");                        \
    }

static int check_dims(int model, int ns, int m) {
    int en = -1, em = -1;
    switch (model) {
        case FCB_MODEL_SINGLE_INTEGRATOR_2D: en = 2; em = 2; break;
        case FCB_MODEL_DIFF_DRIVE: en = 3; em = 2; break;
        case FCB_MODEL_AIRCRAFT_3D: en = 6; em = 3; break;
        case FCB_MODEL_DOUBLE_INTEGRATOR_2D: en = 4; em = 2; break;
        case FCB_MODEL_LTI: return (ns >= 1 && ns <= 6 && m >= 1 && m <= 3)
                                       ? FCB_OK
                                       : fail(FCB_ENOTSUP, "LTI model needs 1<=ns<=6, 1<=m<=3");
        default: return fail(FCB_ENOTSUP, "unknown device model id");
    }
    if (ns != en || m != em) return fail(FCB_EINPUT, "state/control dims do not match the model");
    return FCB_OK;
}

// Phi = I + hA + (hA)^2/2 + (hA)^3/6 + (hA)^4/24, Gam = h (I + hA/2 + (hA)^2/6
// + (hA)^3/24) B: one RK4/ZOH step of a linear model as an affine map.
template <class Mdl>
__device__ void phigam_compute(const double* prm, double dt, double* out) {
    constexpr int N = Mdl::N, M = Mdl::M;
    double A[N * N], B[N * M], z0[N] = {}, u0[M] = {};
    Mdl::jac(z0, u0, prm, A, B);
    double hA[N][N], Pw[N][N], Phi[N][N], Gs[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            hA[i][j] = dt * A[i * N + j];
            Pw[i][j] = Phi[i][j] = Gs[i][j] = (i == j) ? 1.0 : 0.0;
        }
    const double cphi[5] = {1.0, 1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0};
    const double cgam[4] = {1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0};
#pragma unroll
    for (int p = 1; p <= 4; ++p) {
        double Nw[N][N];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) {
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < N; ++q) s += Pw[i][q] * hA[q][j];
                Nw[i][j] = s;
            }
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) {
                Pw[i][j] = Nw[i][j];
                Phi[i][j] += cphi[p] * Pw[i][j];
                if (p <= 3) Gs[i][j] += cgam[p] * Pw[i][j];
            }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) out[i * N + j] = Phi[i][j];
#pragma unroll
        for (int j = 0; j < M; ++j) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += Gs[i][q] * B[q * M + j];
            out[N * N + i * M + j] = dt * s;
        }
    }
}

template <class Mdl>
__global__ void phigam_kernel(const double* prm, double dt, double* out, const int* gate) {
    if (threadIdx.x != 0) return;
    if (gate && *((volatile const int*)gate) != 0) return;
    phigam_compute<Mdl>(prm, dt, out);
}

// One-launch rollouts for T <= AS_BLK^2 (fused_scan): Phi/Gam, the scan with
// the fused state/workspace outputs, and the status epilogue (block 0 takes
// the first non-finite step over all blocks).
__device__ __forceinline__ void roll_publish_and_finish(const FusedWs& fw, unsigned* flags,
                                                        unsigned tag, int first_bad, int* s_min,
                                                        int* status, int* plan_state,
                                                        int iteration) {
    const int t = threadIdx.x, nb = gridDim.x;
    if (t == 0) {
        fw.ivals[blockIdx.x] = first_bad;
        __threadfence();
        st_release_flag(flags + blockIdx.x, tag);
    }
    if (blockIdx.x != 0) return;
    if (t == 0) *s_min = 0x7f7f7f7f;
    __syncthreads();
    if (t < nb) {
        wait_flag(flags, t, tag);
        atomicMin(s_min, __ldcg(fw.ivals + t));
    }
    __syncthreads();
    if (t == 0) roll_finish_body(*s_min, status, plan_state, iteration);
}

template <class Mdl>
__global__ void __launch_bounds__(AS_BLK)
    roll_fused_linear_kernel(const double* prm, double dt, const double* s0, const double* U, int T,
                             double* S, int d, const double* P, double* X, int* status,
                             int* plan_state, int iteration, FusedWs fw, unsigned tag) {
    constexpr int N = Mdl::N, M = Mdl::M;
    extern __shared__ double sbuf[];
    __shared__ ScanShared<N> sh;
    __shared__ double pg[N * N + N * M];
    __shared__ int first_bad, s_min;
    if (plan_state && *((volatile int*)plan_state) != 0) return;
    if (threadIdx.x == 0) {
        phigam_compute<Mdl>(prm, dt, pg);
        first_bad = 0x7f7f7f7f;
    }
    __syncthreads();
    RollMap<N, M> mapf{pg, U};
    RollOut<Mdl> out{S, s0, X, P, d, &first_bad, prm, U, dt};
    fused_scan<N, true>(T, mapf, out, s0, fw.agg0, fw.flags, tag, sbuf, sh);
    roll_publish_and_finish(fw, fw.flags + AS_BLK, tag, first_bad, &s_min, status, plan_state,
                            iteration);
}

template <class Mdl>
__global__ void __launch_bounds__(AS_BLK)
    roll_fused_tri_kernel(const double* s0, const double* U, int T, double dt, double* S, int d,
                          const double* P, double* X, double* dp, int* status, int* plan_state,
                          int iteration, FusedWs fw, unsigned tag) {
    extern __shared__ double sbuf[];
    __shared__ ScanShared<Mdl::NQ> shq;
    __shared__ ScanShared<Mdl::NP> shp;
    __shared__ int first_bad, s_min;
    if (plan_state && *((volatile int*)plan_state) != 0) return;
    if (threadIdx.x == 0) first_bad = 0x7f7f7f7f;
    __syncthreads();
    TriQMap<Mdl> qmap{U, dt};
    TriQOut<Mdl> qout{U, dt, S, s0, dp, &first_bad};
    fused_scan<Mdl::NQ, true>(T, qmap, qout, s0 + Mdl::QOFF, fw.agg0, fw.flags, tag, sbuf, shq);
    TriPMap<Mdl> pmap{dp};
    TriPOut<Mdl> pout{S, X, P, d, &first_bad};
    fused_scan<Mdl::NP, true>(T, pmap, pout, s0, fw.agg1, fw.flags + AS_BLK, tag, sbuf, shp);
    roll_publish_and_finish(fw, fw.flags + 2 * AS_BLK, tag, first_bad, &s_min, status, plan_state,
                            iteration);
}

static std::atomic<unsigned> g_scan_tag{0x5eed0000u};
unsigned next_scan_tag() { return g_scan_tag.fetch_add(1u, std::memory_order_relaxed); }

static FusedWs fused_take(Arena& ar) {
    FusedWs f{};
    f.agg0 = ar.take<double>(fused_agg_doubles<6>());
    f.agg1 = ar.take<double>(fused_agg_doubles<6>());
    f.vals = ar.take<double>(FUSED_MAX_BLOCKS);
    f.ivals = ar.take<int>(FUSED_MAX_BLOCKS);
    f.flags = ar.take<unsigned>(4 * AS_BLK);
    return f;
}

// dynamic shared memory of a fused kernel (the in-block scan buffers)
template <class Kern>
static size_t fused_smem(Kern k, size_t bytes) {
    static size_t set = 0;  // per kernel instantiation
    if (bytes > set) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        set = bytes;
    }
    return bytes;
}

struct RollWs {
    double* phigam;
    double* scan;
    double* dp;
    int* first_bad;
    FusedWs fw;
    size_t bytes;
};

static RollWs roll_layout(int ns, int T, void* ws) {
    Arena ar(ws, ws ? (size_t)-1 : 0);
    RollWs L{};
    L.phigam = ar.take<double>(6 * 6 + 6 * 3);
    L.scan = ar.take<double>(affscan_scratch_doubles<6>(T));  // sized for the largest N
    L.dp = ar.take<double>((size_t)T * 3);                    // triangular models' increments
    L.first_bad = ar.take<int>(4);
    L.fw = fused_take(ar);
    L.bytes = ar.off + 256;
    (void)ns;
    return L;
}

size_t rollout_ws_bytes(int ns, int T) { return roll_layout(ns, T, nullptr).bytes; }

template <class Mdl>
static int launch_rollout(int method, const double* prm, const double* s0, const double* U, int T,
                          double dt, double* S, int d, const double* P, double* X, int* status,
                          int* plan_state, int iteration, double* ws, cudaStream_t st) {
    constexpr int N = Mdl::N, M = Mdl::M;
    if constexpr (Mdl::LINEAR) {
        if (method == 1 && ws != nullptr && fused_scan_ok(T)) {
            RollWs L = roll_layout(N, T, ws);
            auto kern = roll_fused_linear_kernel<Mdl>;
            const size_t smem = fused_smem(kern, fused_smem_bytes<N>());
            kern<<<fused_blocks(T), AS_BLK, smem, st>>>(prm, dt, s0, U, T, S, d, P, X, status,
                                                          plan_state, iteration, L.fw,
                                                          next_scan_tag());
            return 1;
        }
    }
    if (Mdl::LINEAR && method == 1 && ws != nullptr) {
        RollWs L = roll_layout(N, T, ws);
        cudaMemsetAsync(L.first_bad, 0x7f, sizeof(int), st);
        phigam_kernel<Mdl><<<1, 32, 0, st>>>(prm, dt, L.phigam, plan_state);
        RollMap<N, M> mapf{L.phigam, U};
        RollOut<Mdl> out{S, s0, X, P, d, L.first_bad, prm, U, dt};
        const int n = affscan_run<N, true>(T, mapf, out, s0, affscan_bufs<N>(L.scan, T),
                                           plan_state, st);
        roll_finish_kernel<<<1, 32, 0, st>>>(L.first_bad, status, plan_state, iteration);
        return n + 2;
    }
    if constexpr (Mdl::TRIANGULAR) {
        if (method == 1 && ws != nullptr && fused_scan_ok(T)) {
            RollWs L = roll_layout(N, T, ws);
            auto kern = roll_fused_tri_kernel<Mdl>;
            constexpr int NMAX = Mdl::NQ > Mdl::NP ? Mdl::NQ : Mdl::NP;
            const size_t smem = fused_smem(kern, fused_smem_bytes<NMAX>());
            kern<<<fused_blocks(T), AS_BLK, smem, st>>>(s0, U, T, dt, S, d, P, X, L.dp, status,
                                                          plan_state, iteration, L.fw,
                                                          next_scan_tag());
            return 1;
        }
        if (method == 1 && ws != nullptr) {
            RollWs L = roll_layout(N, T, ws);
            cudaMemsetAsync(L.first_bad, 0x7f, sizeof(int), st);
            TriQMap<Mdl> qmap{U, dt};
            TriQOut<Mdl> qout{U, dt, S, s0, L.dp, L.first_bad};
            int n = affscan_run<Mdl::NQ, true>(T, qmap, qout, s0 + Mdl::QOFF,
                                               affscan_bufs<Mdl::NQ>(L.scan, T), plan_state, st);
            TriPMap<Mdl> pmap{L.dp};
            TriPOut<Mdl> pout{S, X, P, d, L.first_bad};
            n += affscan_run<Mdl::NP, true>(T, pmap, pout, s0, affscan_bufs<Mdl::NP>(L.scan, T),
                                            plan_state, st);
            roll_finish_kernel<<<1, 32, 0, st>>>(L.first_bad, status, plan_state, iteration);
            return n + 1;
        }
    }
    rollout_kernel<Mdl><<<1, 32, 0, st>>>(prm, s0, U, T, dt, S, d, P, X, status, plan_state,
                                          iteration);
    return 1;
}

int rollout(int model, int ns, int m, const double* prm, const double* s0, const double* U, int T,
            double dt, double* S, int d, const double* P, double* X, int* status, int* plan_state,
            int iteration, int method, double* ws, cudaStream_t st) {
    int rc = check_dims(model, ns, m);
    if (rc) return rc;
    if (T < 1) return fail(FCB_EINPUT, "need at least one control step");
    int launches = 0;
    FCB_MODEL_DISPATCH((launches = launch_rollout<Mdl>(method, prm, s0, U, T, dt, S, d, P, X,
                                                       status, plan_state, iteration, ws, st)));
    count_launch(launches - 1);
    FCB_LAUNCHED("rollout_kernel");
    return FCB_OK;
}

int linearize(int model, int ns, int m, const double* prm, const double* S, const double* U, int T,
              double* A, double* B, cudaStream_t st) {
    int rc = check_dims(model, ns, m);
    if (rc) return rc;
    if (T < 1) return FCB_OK;
    const int blocks = std::min(4 * sm_count(), (T + 127) / 128);
    FCB_MODEL_DISPATCH((linearize_kernel<Mdl><<<blocks, 128, 0, st>>>(prm, S, U, T, A, B)));
    FCB_LAUNCHED("linearize_kernel");
    return FCB_OK;
}

// Workspace of the two-phase LQR: Riccati scan aggregates, per-step Riccati
// outputs (K, H^-1 G', Acl, G; element-major), d, the affine-scan scratch, a
// status word and the one-launch scan flags.
struct LqrWs {
    RicGeom geom;
    double *agg, *bagg, *K, *Lg, *Acl, *Gm, *dff, *scan;
    int* fail;
    FusedWs fw;
    size_t bytes;
};

static LqrWs lqr_layout(int ns, int m, int T, void* ws) {
    Arena ar(ws, ws ? (size_t)-1 : 0);
    LqrWs L{};
    L.geom = ric_geom(T, ric_max_blocks());
    L.agg = ar.take<double>(2 * (size_t)L.geom.nwarp * 3 * ns * ns);
    L.bagg = ar.take<double>((2 * (size_t)L.geom.nblk + 2 * RW_K2_WARPS) * 3 * ns * ns);
    L.K = ar.take<double>((size_t)T * m * ns);
    L.Lg = ar.take<double>((size_t)T * m * ns);
    L.Acl = ar.take<double>((size_t)T * ns * ns);
    L.Gm = ar.take<double>((size_t)T * ns * m);
    L.dff = ar.take<double>((size_t)T * m);
    L.scan = ar.take<double>(affscan_scratch_doubles<6>(T));
    L.fail = ar.take<int>(4);
    L.fw = fused_take(ar);
    L.bytes = ar.off + 256;
    return L;
}

size_t lqr_ws_bytes(int ns, int m, int T) { return lqr_layout(ns, m, T, nullptr).bytes; }

static RicArgs ric_args(const LqrWs& L, int T, double dt, const double* Q, const double* R) {
    RicArgs r{};
    r.T = T;
    r.dt = dt;
    r.Q = Q;
    r.R = R;
    r.agg = L.agg;
    r.bagg = L.bagg;
    r.L = L.geom.L;
    r.nwarp = L.geom.nwarp;
    r.nblk = L.geom.nblk;
    r.K = L.K;
    r.Lg = L.Lg;
    r.Acl = L.Acl;
    r.Gm = L.Gm;
    r.fail = L.fail;
    return r;
}

// The affine phase: eta (backward scan, emits d), z (forward scan: v*, cost,
// z, U update), then the finish kernel.  Returns the number of launches.
template <int N, int M, class Flow>
static int affine_phase(const LqrWs& L, const double* K, double* dff, int T, double dt,
                        const double* Q, const double* R, const Flow& flow, double* v, double* z,
                        const double* U, double* U_next, double eta, const double* clamp,
                        double* cost, double* lqr_costs, int* plan_state, int iteration,
                        int reset_fail, cudaStream_t st) {
    EtaMap<N, Flow> emap{L.Acl, Q, dt, T, flow};
    EtaOut<N, M> eout{L.Lg, dff, L.fail, T};
    ZMap<N, M> zmap{L.Acl, L.Gm, dff, T};
    ZOut<N, M, Flow> zout{K, T, dff, Q, R, dt, flow, L.fail, v, z, U, U_next, eta, clamp};
    if (fused_scan_ok(T)) {
        auto kern = affine_fused_kernel<N, M, Flow>;
        const size_t smem = fused_smem(kern, fused_smem_bytes<N>());
        kern<<<fused_blocks(T), AS_BLK, smem, st>>>(T, emap, eout, zmap, zout, L.fw,
                                                      next_scan_tag(), L.fail, reset_fail, cost,
                                                      lqr_costs, plan_state, iteration);
        return 1;
    }
    if (reset_fail) cudaMemsetAsync(L.fail, 0xff, sizeof(int), st);
    const AffScanBufs b = affscan_bufs<N>(L.scan, T);
    int n = affscan_run<N, false>(T, emap, eout, nullptr, b, plan_state, st);
    n += affscan_run<N, true>(T, zmap, zout, nullptr, b, plan_state, st);
    lqr_finish_kernel<<<1, 32, 0, st>>>(affscan_blocks(T), b.red, L.fail, cost, lqr_costs,
                                        plan_state, iteration, plan_state != nullptr);
    return n + 1;
}

// X[e * T + k] -> Y[k * E + e]
__global__ void step_major_kernel(const double* __restrict__ X, int T, int E,
                                  double* __restrict__ Y) {
    const size_t n = (size_t)T * E;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const size_t k = i / E, e = i % E;
        Y[i] = X[e * T + k];
    }
}

template <int N, int M>
static int lqr_solve_t(int T, double dt, const double* A, const double* B, const double* Q,
                       const double* R, const double* a, double* v, double* z, double* K,
                       double* dff, double* scal, const LqrWs& L, cudaStream_t st) {
    RicArgs r = ric_args(L, T, dt, Q, R);
    const int nr = ric_phase<N, M>(ric_arrays_k1<N, M>, ric_arrays_k3<N, M>, r, st, false, A, B);
    ArrayFlow<N> fl{a};
    int n = nr + affine_phase<N, M>(L, L.K, dff ? dff : L.dff, T, dt, Q, R, fl, v, z, nullptr,
                                   nullptr, 0.0, nullptr, scal, nullptr, nullptr, 0, 0, st);
    if (K) {  // gains to the caller's step-major layout [T][M][N]
        const int blocks = std::min(4 * sm_count(), (T * M * N + 255) / 256);
        step_major_kernel<<<blocks, 256, 0, st>>>(L.K, T, M * N, K);
        ++n;
    }
    return n;
}

int lqr_solve(int ns, int m, int T, double dt, const double* A, const double* B, const double* Q,
              const double* R, const double* a, double* v, double* z, double* K, double* dff,
              double* scal, int* status, double* ws, cudaStream_t st) {
    if (T < 1) return fail(FCB_EINPUT, "horizon must be >= 1");
    if (!ws) return fail(FCB_EWORKSPACE, "lqr needs a workspace (fcb_lqr_workspace_bytes)");
    LqrWs L = lqr_layout(ns, m, T, ws);
    int n = 0;
#define FCB_LQR_CASE(NN, MM)                                                                  \
    case NN * 4 + MM:                                                                         \
        n = lqr_solve_t<NN, MM>(T, dt, A, B, Q, R, a, v, z, K, dff, scal, L, st);             \
        break;
    switch (ns * 4 + m) {
        FCB_LQR_CASE(1, 1) FCB_LQR_CASE(1, 2) FCB_LQR_CASE(1, 3)
        FCB_LQR_CASE(2, 1) FCB_LQR_CASE(2, 2) FCB_LQR_CASE(2, 3)
        FCB_LQR_CASE(3, 1) FCB_LQR_CASE(3, 2) FCB_LQR_CASE(3, 3)
        FCB_LQR_CASE(4, 1) FCB_LQR_CASE(4, 2) FCB_LQR_CASE(4, 3)
        FCB_LQR_CASE(5, 1) FCB_LQR_CASE(5, 2) FCB_LQR_CASE(5, 3)
        FCB_LQR_CASE(6, 1) FCB_LQR_CASE(6, 2) FCB_LQR_CASE(6, 3)
        default: return fail(FCB_ENOTSUP, "lqr needs 1<=n<=6 and 1<=m<=3");
    }
#undef FCB_LQR_CASE
    count_launch(n - 1);
    FCB_LAUNCHED("lqr_scan_kernels");
    FCB_CUDA(cudaMemcpyAsync(status, L.fail, sizeof(int), cudaMemcpyDeviceToDevice, st));
    return FCB_OK;
}

size_t plan_update_ws_bytes(int ns, int m, int T) { return lqr_ws_bytes(ns, m, T); }

template <class Mdl>
static int launch_plan_update(int mode, const LqrWs& L, int T, double dt, const double* Q,
                              const double* R, const double* prm, const double* S, const double* U,
                              const double* flow, const double* P, int d, double eta,
                              const double* clamp, double* Unext, double* lqr_costs,
                              int* plan_state, int iteration, cudaStream_t st) {
    constexpr int N = Mdl::N, M = Mdl::M;
    int n = 0;
    if (mode != 1) {
        RicArgs r = ric_args(L, T, dt, Q, R);
        r.plan_state = plan_state;
        r.iteration = iteration;
        n = ric_phase<N, M>(plan_ric_k1<Mdl>, plan_ric_k3<Mdl>, r, st, true, prm, S, U);
    }
    // mode 1: fail := -1, the stored Riccati phase is valid
    LiftedFlow<N> fl{flow, P, d};
    return n + affine_phase<N, M>(L, L.K, L.dff, T, dt, Q, R, fl, nullptr, nullptr, U, Unext, eta,
                                  clamp, nullptr, lqr_costs, plan_state, iteration, mode == 1, st);
}

int plan_update(int model, int ns, int m, const double* prm, const double* S, const double* U,
                int T, double dt, int d, const double* P, const double* flow, const double* Q,
                const double* R, double eta, const double* clamp, double* Unext, double* lqr_costs,
                int* plan_state, int iteration, int mode, double* ws, size_t ws_bytes,
                cudaStream_t st) {
    int rc = check_dims(model, ns, m);
    if (rc) return rc;
    if (ws_bytes < plan_update_ws_bytes(ns, m, T))
        return fail(FCB_EWORKSPACE, "plan_update workspace too small");
    LqrWs L = lqr_layout(ns, m, T, ws);
    int n = 0;
    FCB_MODEL_DISPATCH((n = launch_plan_update<Mdl>(mode, L, T, dt, Q, R, prm, S, U, flow, P, d,
                                                    eta, clamp, Unext, lqr_costs, plan_state,
                                                    iteration, st)));
    count_launch(n - 1);
    FCB_LAUNCHED("plan_update_kernels");
    return FCB_OK;
}

// ---------------------------------------------------------------------------
// the fused planner loop (plan_fused.cuh)
// ---------------------------------------------------------------------------
}  // namespace fcb
#include "plan_fused.cuh"
#include "plan_stein.cuh"
namespace fcb {

struct PfWs {
    RsWs rs;
    double* agg;
    double* part;
    int* ipart;
    double* dff;
    size_t total;
};

static PfWs pf_layout(int batch, int n, int m, int d, int mc, int group, void* ws, size_t bytes) {
    PfWs L{};
    L.rs = rs_layout(batch, n, m, d, group, ws, bytes);
    Arena ar(ws ? (char*)ws + L.rs.total : nullptr, ws ? (bytes > L.rs.total ? bytes - L.rs.total : 0) : 0);
    L.agg = ar.take<double>((size_t)2 * PF_CARRY * (6 * 6 + 6));
    L.part = ar.take<double>(PF_CARRY);
    L.ipart = ar.take<int>(PF_CARRY);
    L.dff = ar.take<double>((size_t)batch * n * mc);
    L.total = L.rs.total + ar.off + 256;
    return L;
}

size_t plan_fused_ws_bytes(int batch, int T, int M, int d, int mc) {
    const int G = batch > 1 ? 1 : sm_count();
    return pf_layout(batch, T, M, d, mc, G, nullptr, 0).total;
}

template <class Mdl, int D, bool GRID>
static int pf_launch(const RsArgs& a, const PlanFusedArgs<Mdl::N, Mdl::M>& pf, int grid,
                     size_t smem, cudaStream_t st) {
    auto kern = rs_plan_kernel<D, GRID, Mdl>;
    static size_t attr = 0;
    if (attr < smem) {
        FCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
    }
    RsArgs ac = a;
    PlanFusedArgs<Mdl::N, Mdl::M> pc = pf;
    if (GRID) {
        void* args[] = {&ac, &pc};
        FCB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(RS_BLOCK), args,
                                             smem, st));
    } else {
        kern<<<grid, RS_BLOCK, smem, st>>>(ac, pc);
    }
    FCB_LAUNCHED("rs_plan_kernel");
    return FCB_OK;
}

template <class Mdl>
static int plan_fused_t(const double* prm, const double* s0, double* U0, double* U1, double* S0,
                        double* S1, int T, double dt, int d, const double* P, double* X,
                        double* flow, const double* Q, const double* R, double eta,
                        const double* clamp, const double* Y, int M, double omega_fixed,
                        int max_iters, double tol, double conv_tol, double* warm_f,
                        double* warm_p, int* warm_valid, double* fstat, int* plan_state,
                        double* flow_log, double* lqr_costs, unsigned long long* phase_ns,
                        int it0, int maxit, int batch, const void* upd_ws, void* ws,
                        size_t ws_bytes, cudaStream_t st) {
    constexpr int N = Mdl::N, MC = Mdl::M;
    if constexpr (!Mdl::LINEAR || N > 4) {
        return fail(FCB_ENOTSUP, "the fused planner needs a linear model with at most 4 states");
    } else {
        const bool grid_mode = batch <= 1;
        const int G = grid_mode ? sm_count() : 1;
        if (G > PF_CARRY) return fail(FCB_ENOTSUP, "too many SMs for the fused planner");
        const RsShape sh = rs_shape(T, M, d, G, grid_mode);
        if (!sh.ok) return fail(FCB_ENOTSUP, "point sets do not fit in shared memory");
        size_t smem = std::max(sh.smem, pf_smem_bytes<N>());
        int const_off = 0;
        if (grid_mode) {  // per-CTA copy of the stored Riccati arrays
            const size_t cmax = (size_t)(T + G - 1) / G;
            const size_t cbytes = cmax * (N * N + 3 * MC * N) * sizeof(double);
            const size_t off = align_up(smem, 16);
            if (off + cbytes + RS_STATIC_SMEM <= (size_t)rs_smem_limit()) {
                const_off = (int)off;
                smem = off + cbytes;
            }
        }
        if (smem + RS_STATIC_SMEM > (size_t)rs_smem_limit())
            return fail(FCB_ENOTSUP, "fused planner shared memory");
        PfWs L = pf_layout(batch, T, M, d, MC, G, ws, ws_bytes);
        if (L.total > ws_bytes) return fail(FCB_EWORKSPACE, "plan_fused workspace too small");
        LqrWs W = lqr_layout(N, MC, T, const_cast<void*>(upd_ws));
        RsArgs a{};
        a.X = X;
        a.Y = Y;
        a.n = T;
        a.m = M;
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
        a.iteration = it0;
        a.flow_log = flow_log;
        a.log_stride = 4LL * maxit;
        rs_fill(a, L.rs, sh);
        a.launch_id = next_launch_epoch();
        PlanFusedArgs<N, MC> pf{};
        pf.T = T;
        pf.d = d;
        pf.it0 = it0;
        pf.maxit = maxit;
        pf.dt = dt;
        pf.eta = eta;
        pf.s0 = s0;
        pf.prm = prm;
        pf.P = P;
        pf.Q = Q;
        pf.R = R;
        pf.clamp = clamp;
        pf.K = W.K;
        pf.Lg = W.Lg;
        pf.Acl = W.Acl;
        pf.Gm = W.Gm;
        pf.dff = L.dff;
        pf.U0 = U0;
        pf.U1 = U1;
        pf.S0 = S0;
        pf.S1 = S1;
        pf.lqr_costs = lqr_costs;
        pf.phase_ns = phase_ns;
        pf.const_off = const_off;
        pf.agg = L.agg;
        pf.part = L.part;
        pf.ipart = L.ipart;
        const int grid = grid_mode ? G : batch;
        // the built-in linear models cover a planar workspace
        if (d != 2) return fail(FCB_ENOTSUP, "the fused planner covers planar workspaces");
        return grid_mode ? pf_launch<Mdl, 2, true>(a, pf, grid, smem, st)
                         : pf_launch<Mdl, 2, false>(a, pf, grid, smem, st);
    }
}

int plan_fused(int model, int ns, int m, const double* prm, const double* s0, double* U0,
               double* U1, double* S0, double* S1, int T, double dt, int d, const double* P,
               double* X, double* flow, const double* Q, const double* R, double eta,
               const double* clamp, const double* Y, int M, double omega_fixed, int max_iters,
               double tol, double conv_tol, double* warm_f, double* warm_p, int* warm_valid,
               double* fstat, int* plan_state, double* flow_log, double* lqr_costs,
               unsigned long long* phase_ns, int it0, int maxit, int batch, const void* upd_ws,
               void* ws, size_t ws_bytes, cudaStream_t st) {
    int rc = check_dims(model, ns, m);
    if (rc) return rc;
    if (d < 1 || d > 3) return fail(FCB_ENOTSUP, "point dimension must be 1, 2 or 3");
    if (it0 >= maxit) return FCB_OK;
    switch (model) {
        case FCB_MODEL_SINGLE_INTEGRATOR_2D:
            return plan_fused_t<Model<FCB_MODEL_SINGLE_INTEGRATOR_2D>>(
                prm, s0, U0, U1, S0, S1, T, dt, d, P, X, flow, Q, R, eta, clamp, Y, M, omega_fixed,
                max_iters, tol, conv_tol, warm_f, warm_p, warm_valid, fstat, plan_state, flow_log,
                lqr_costs, phase_ns, it0, maxit, batch, upd_ws, ws, ws_bytes, st);
        case FCB_MODEL_DOUBLE_INTEGRATOR_2D:
            return plan_fused_t<Model<FCB_MODEL_DOUBLE_INTEGRATOR_2D>>(
                prm, s0, U0, U1, S0, S1, T, dt, d, P, X, flow, Q, R, eta, clamp, Y, M, omega_fixed,
                max_iters, tol, conv_tol, warm_f, warm_p, warm_valid, fstat, plan_state, flow_log,
                lqr_costs, phase_ns, it0, maxit, batch, upd_ws, ws, ws_bytes, st);
        default:
            return fail(FCB_ENOTSUP, "the fused planner supports the built-in linear models");
    }
}

// ---------------------------------------------------------------------------
// the fused SVGD planner loop (plan_stein.cuh)
// ---------------------------------------------------------------------------
struct SfpWs {
    GridBarrier* bar;
    unsigned* done;
    double* agg;
    double* part;
    int* ipart;
    double* dff;
    double* scores;
    unsigned* hist;
    unsigned long long* cand;
    unsigned* ccount;
    double* npart;
    size_t total;
};

static SfpWs sfp_layout(int T, int d, int mc, void* ws, size_t bytes) {
    Arena ar(ws, bytes);
    SfpWs L{};
    L.bar = ar.take<GridBarrier>(1);
    L.done = ar.take<unsigned>(32);
    L.agg = ar.take<double>((size_t)2 * PF_CARRY * (6 * 6 + 6));
    L.part = ar.take<double>(PF_CARRY);
    L.ipart = ar.take<int>(PF_CARRY);
    L.dff = ar.take<double>((size_t)T * mc);
    L.scores = ar.take<double>((size_t)T * d);
    L.hist = ar.take<unsigned>((size_t)3 * 2 * SVP_BINS);
    L.cand = ar.take<unsigned long long>(SVP_CAND);
    L.ccount = ar.take<unsigned>(2);
    L.npart = ar.take<double>(PF_CARRY);
    L.total = ar.off + 256;
    return L;
}

size_t plan_stein_ws_bytes(int T, int d, int mc) { return sfp_layout(T, d, mc, nullptr, 0).total; }

template <class Mdl, int D>
static int sfp_launch(const SvFusedArgs<Mdl::N, Mdl::M>& a, int grid, size_t smem,
                      cudaStream_t st) {
    auto kern = sv_plan_kernel<D, Mdl>;
    cudaFuncAttributes fa{};
    FCB_CUDA(cudaFuncGetAttributes(&fa, (const void*)kern));
    if (fa.sharedSizeBytes + smem > (size_t)rs_smem_limit())
        return fail(FCB_ENOTSUP, "fused Stein planner shared memory");
    static size_t granted = 0;
    if (granted < smem) {
        FCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        granted = smem;
    }
    int per_sm = 0;
    FCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RS_BLOCK, smem));
    if (per_sm < 1) return fail(FCB_ENOTSUP, "fused Stein planner not co-resident");
    SvFusedArgs<Mdl::N, Mdl::M> ac = a;
    void* args[] = {&ac};
    FCB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(RS_BLOCK), args, smem,
                                         st));
    FCB_LAUNCHED("sv_plan_kernel");
    return FCB_OK;
}

template <class Mdl>
static int plan_stein_t(const double* prm, const double* s0, double* U0, double* U1, double* S0,
                        double* S1, int T, double dt, int d, const double* P, double* X,
                        double* flow, const double* Q, const double* R, double eta,
                        const double* clamp, int k, const double* gmm, double bw_fixed,
                        double log_np1, double conv_tol, double* fstat, int* plan_state,
                        double* flow_log, double* lqr_costs, unsigned long long* phase_ns,
                        int it0, int maxit, const void* upd_ws, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
    constexpr int N = Mdl::N, MC = Mdl::M;
    if constexpr (!Mdl::LINEAR || N > 4) {
        return fail(FCB_ENOTSUP, "the fused planner needs a linear model with at most 4 states");
    } else {
        const int G = sm_count();
        if (G > PF_CARRY) return fail(FCB_ENOTSUP, "too many SMs for the fused planner");
        if (d != 2) return fail(FCB_ENOTSUP, "the fused planner covers planar workspaces");
        if ((T + G - 1) / G > 64 || T < 2)
            return fail(FCB_ENOTSUP, "fused Stein planner: 2 <= T <= 64 x SMs");
        // dynamic smem: scan scratch | this CTA's Riccati arrays | the column set
        const size_t cmax = (size_t)(T + G - 1) / G;
        const int const_off = (int)align_up(pf_smem_bytes<N>(), 16);
        const size_t cbytes = cmax * (N * N + 3 * MC * N) * sizeof(double);
        const int sv_off = (int)align_up(const_off + cbytes, 16);
        const size_t smem = sv_off + (size_t)2 * T * d * sizeof(double);
        SfpWs L = sfp_layout(T, d, MC, ws, ws_bytes);
        if (L.total > ws_bytes) return fail(FCB_EWORKSPACE, "fused Stein workspace too small");
        LqrWs W = lqr_layout(N, MC, T, const_cast<void*>(upd_ws));
        FCB_CUDA(cudaMemsetAsync(L.hist, 0, (size_t)3 * 2 * SVP_BINS * sizeof(unsigned), st));
        FCB_CUDA(cudaMemsetAsync(L.ccount, 0, 2 * sizeof(unsigned), st));
        SvFusedArgs<N, MC> a{};
        PlanFusedArgs<N, MC>& pf = a.pf;
        pf.T = T;
        pf.d = d;
        pf.it0 = it0;
        pf.maxit = maxit;
        pf.dt = dt;
        pf.eta = eta;
        pf.s0 = s0;
        pf.prm = prm;
        pf.P = P;
        pf.Q = Q;
        pf.R = R;
        pf.clamp = clamp;
        pf.K = W.K;
        pf.Lg = W.Lg;
        pf.Acl = W.Acl;
        pf.Gm = W.Gm;
        pf.dff = L.dff;
        pf.U0 = U0;
        pf.U1 = U1;
        pf.S0 = S0;
        pf.S1 = S1;
        pf.lqr_costs = lqr_costs;
        pf.phase_ns = phase_ns;
        pf.const_off = const_off;
        pf.agg = L.agg;
        pf.part = L.part;
        pf.ipart = L.ipart;
        a.X = X;
        a.flow = flow;
        a.scores = L.scores;
        a.gmm = gmm;
        a.k = k;
        a.bw_fixed = bw_fixed;
        a.log_np1 = log_np1;
        a.conv_tol = conv_tol;
        a.fstat = fstat;
        a.plan_state = plan_state;
        a.flow_log = flow_log;
        a.hist = L.hist;
        a.cand = L.cand;
        a.ccount = L.ccount;
        a.npart = L.npart;
        a.bar = L.bar;
        a.done = L.done;
        a.launch_id = next_launch_epoch();
        a.sv_off = sv_off;
        return sfp_launch<Mdl, 2>(a, G, smem, st);
    }
}

int plan_stein(int model, int ns, int m, const double* prm, const double* s0, double* U0,
               double* U1, double* S0, double* S1, int T, double dt, int d, const double* P,
               double* X, double* flow, const double* Q, const double* R, double eta,
               const double* clamp, int k, const double* gmm, double bw_fixed, double log_np1,
               double conv_tol, double* fstat, int* plan_state, double* flow_log,
               double* lqr_costs, unsigned long long* phase_ns, int it0, int maxit,
               const void* upd_ws, void* ws, size_t ws_bytes, cudaStream_t st) {
    int rc = check_dims(model, ns, m);
    if (rc) return rc;
    if (it0 >= maxit) return FCB_OK;
    if (k < 1) return fail(FCB_EINPUT, "mixture needs at least one component");
    switch (model) {
        case FCB_MODEL_SINGLE_INTEGRATOR_2D:
            return plan_stein_t<Model<FCB_MODEL_SINGLE_INTEGRATOR_2D>>(
                prm, s0, U0, U1, S0, S1, T, dt, d, P, X, flow, Q, R, eta, clamp, k, gmm, bw_fixed,
                log_np1, conv_tol, fstat, plan_state, flow_log, lqr_costs, phase_ns, it0, maxit,
                upd_ws, ws, ws_bytes, st);
        case FCB_MODEL_DOUBLE_INTEGRATOR_2D:
            return plan_stein_t<Model<FCB_MODEL_DOUBLE_INTEGRATOR_2D>>(
                prm, s0, U0, U1, S0, S1, T, dt, d, P, X, flow, Q, R, eta, clamp, k, gmm, bw_fixed,
                log_np1, conv_tol, fstat, plan_state, flow_log, lqr_costs, phase_ns, it0, maxit,
                upd_ws, ws, ws_bytes, st);
        default:
            return fail(FCB_ENOTSUP, "the fused planner supports the built-in linear models");
    }
}

}  // namespace fcb

// Debug (FCB_TIMELINE builds): CTA 0 phase stamps of the fused planner.
extern "C" FCB_API int fcb_debug_plan_timeline(unsigned long long* host_out, int cap) {
#ifdef FCB_TIMELINE
    unsigned n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, fcb::g_rs_tl_n, sizeof(unsigned));
    const int k = (int)std::min<unsigned>(n, (unsigned)cap);
    if (k) cudaMemcpyFromSymbol(host_out, fcb::g_rs_tl, k * sizeof(unsigned long long));
    const unsigned zero = 0;
    cudaMemcpyToSymbol(fcb::g_rs_tl_n, &zero, sizeof(unsigned));
    return k;
#else
    (void)host_out;
    (void)cap;
    return -1;
#endif
}

// Debug: per-block stamps of the last one-launch scan (FCB_SCAN_TL builds).
extern "C" FCB_API int fcb_debug_scan_timeline(unsigned long long* host_out) {
#ifdef FCB_SCAN_TL
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(host_out, fcb::g_scan_tl, sizeof(fcb::g_scan_tl));
    return fcb::AS_BLK * 16;
#else
    (void)host_out;
    return 0;
#endif
}
