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

#include <algorithm>

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

template <class Mdl>
__global__ void rollout_kernel(const double* __restrict__ prm, const double* __restrict__ s0,
                               const double* __restrict__ U, int T, double dt,
                               double* __restrict__ S, int d, const double* __restrict__ P,
                               double* __restrict__ X, int* status, int* plan_state, int iteration) {
    constexpr int N = Mdl::N, M = Mdl::M;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (plan_state && *((volatile int*)plan_state) != 0) return;
    double s[N], u[M], k1[N], k2[N], k3[N], k4[N], tmp[N];
    const double half = DMUL(0.5, dt);
    const double sixth = dt / 6.0;
    for (int j = 0; j < N; ++j) {
        s[j] = s0[j];
        S[j] = s[j];
    }
    int fail_step = -1;
    for (int k = 0; k < T; ++k) {
        for (int j = 0; j < M; ++j) u[j] = U[(size_t)k * M + j];
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
            fail_step = k + 1;
            break;
        }
        for (int j = 0; j < N; ++j) S[(size_t)(k + 1) * N + j] = s[j];
        if (X) {
            for (int r = 0; r < d; ++r) {
                double a = 0.0;
                for (int j = 0; j < N; ++j) a = DADD(a, DMUL(s[j], P[r * N + j]));
                X[(size_t)k * d + r] = a;
            }
        }
    }
    if (status) *status = fail_step;
    if (plan_state && fail_step >= 0) {
        plan_state[FCB_STATE_STOP] = 2;
        plan_state[FCB_STATE_STAGE] = 1;
        plan_state[FCB_STATE_ITER] = iteration;
        plan_state[FCB_STATE_INDEX] = fail_step;
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
// Solve H X = R (H: m x m, R: m x c) by Gaussian elimination with partial
// pivoting (the LAPACK gesv algorithm np.linalg.solve uses).
template <int M, int C>
__device__ __forceinline__ void solve_small(double (&H)[M][M], double (&R)[M][C]) {
#pragma unroll
    for (int col = 0; col < M; ++col) {
        int piv = col;
        double best = fabs(H[col][col]);
#pragma unroll
        for (int r = col + 1; r < M; ++r)
            if (fabs(H[r][col]) > best) {
                best = fabs(H[r][col]);
                piv = r;
            }
        if (piv != col) {
#pragma unroll
            for (int k = 0; k < M; ++k) {
                double t = H[col][k];
                H[col][k] = H[piv][k];
                H[piv][k] = t;
            }
#pragma unroll
            for (int k = 0; k < C; ++k) {
                double t = R[col][k];
                R[col][k] = R[piv][k];
                R[piv][k] = t;
            }
        }
#pragma unroll
        for (int r = col + 1; r < M; ++r) {
            const double l = H[r][col] / H[col][col];
#pragma unroll
            for (int k = col; k < M; ++k) H[r][k] -= l * H[col][k];
#pragma unroll
            for (int k = 0; k < C; ++k) R[r][k] -= l * R[col][k];
        }
    }
#pragma unroll
    for (int r = M - 1; r >= 0; --r) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
            double v = R[r][k];
#pragma unroll
            for (int q = r + 1; q < M; ++q) v -= H[r][q] * R[q][k];
            R[r][k] = v / H[r][r];
        }
    }
}

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

template <int N, int M, class Jac, class Flow>
__device__ void lqr_core(const Jac& jac, const Flow& flow, int T, double dt,
                         const double* __restrict__ Qm, const double* __restrict__ Rm,
                         double* __restrict__ Kout, double* __restrict__ dout,
                         double* __restrict__ v, double* __restrict__ z, double* cost_out,
                         int* fail_out) {
    double Qb[N][N], Rb[M][M];
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) Qb[i][j] = dt * Qm[i * N + j];
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) Rb[i][j] = dt * Rm[i * M + j];
    double P[N][N], p[N];
    for (int i = 0; i < N; ++i) {
        p[i] = 0.0;
        for (int j = 0; j < N; ++j) P[i][j] = 0.0;
    }
    int fail = -1;
    for (int k = T - 1; k >= 0; --k) {
        double a[N * N], b[N * M], ak[N];
        jac.get(k, a, b);
        flow.get(k, ak);
        double F[N][N], G[N][M];
        for (int i = 0; i < N; ++i) {
            for (int j = 0; j < N; ++j) F[i][j] = (i == j ? 1.0 : 0.0) + dt * a[i * N + j];
            for (int j = 0; j < M; ++j) G[i][j] = dt * b[i * M + j];
        }
        double PG[N][M], PF[N][N];
        for (int i = 0; i < N; ++i) {
            for (int j = 0; j < M; ++j) {
                double s = 0.0;
                for (int q = 0; q < N; ++q) s += P[i][q] * G[q][j];
                PG[i][j] = s;
            }
            for (int j = 0; j < N; ++j) {
                double s = 0.0;
                for (int q = 0; q < N; ++q) s += P[i][q] * F[q][j];
                PF[i][j] = s;
            }
        }
        double H[M][M], rhs[M][N + 1];
        for (int i = 0; i < M; ++i) {
            for (int j = 0; j < M; ++j) {
                double s = 0.0;
                for (int q = 0; q < N; ++q) s += G[q][i] * PG[q][j];
                H[i][j] = Rb[i][j] + s;
            }
            for (int j = 0; j < N; ++j) {
                double s = 0.0;
                for (int q = 0; q < N; ++q) s += G[q][i] * PF[q][j];
                rhs[i][j] = s;
            }
            double s = 0.0;
            for (int q = 0; q < N; ++q) s += G[q][i] * p[q];
            rhs[i][N] = -s;
        }
        solve_small<M, N + 1>(H, rhs);
        for (int i = 0; i < M; ++i) {
            for (int j = 0; j < N; ++j) Kout[((size_t)k * M + i) * N + j] = rhs[i][j];
            dout[(size_t)k * M + i] = rhs[i][N];
        }
        double FGK[N][N];
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                double s = 0.0;
                for (int q = 0; q < M; ++q) s += G[i][q] * rhs[q][j];
                FGK[i][j] = F[i][j] - s;
            }
        double PFGK[N][N];
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                double s = 0.0;
                for (int q = 0; q < N; ++q) s += P[i][q] * FGK[q][j];
                PFGK[i][j] = s;
            }
        double Pn[N][N];
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                double s = 0.0;
                for (int q = 0; q < N; ++q) s += F[q][i] * PFGK[q][j];
                Pn[i][j] = Qb[i][j] + s;
            }
        bool finite = true;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                P[i][j] = 0.5 * (Pn[i][j] + Pn[j][i]);
                finite = finite && isfinite(P[i][j]);
            }
        double pn[N];
        for (int i = 0; i < N; ++i) {
            double qa = 0.0;
            for (int q = 0; q < N; ++q) qa += Qb[i][q] * ak[q];
            double s = 0.0;
            for (int q = 0; q < N; ++q) s += FGK[q][i] * p[q];
            pn[i] = -qa + s;
        }
        for (int i = 0; i < N; ++i) {
            p[i] = pn[i];
            finite = finite && isfinite(p[i]);
        }
        if (!finite) {
            fail = k;
            break;
        }
    }
    if (fail_out) *fail_out = fail;
    if (fail >= 0) return;
    double zz[N];
    for (int i = 0; i < N; ++i) {
        zz[i] = 0.0;
        if (z) z[i] = 0.0;
    }
    double cost = 0.0;
    for (int k = 0; k < T; ++k) {
        double a[N * N], b[N * M], ak[N];
        jac.get(k, a, b);
        flow.get(k, ak);
        double vk[M];
        for (int i = 0; i < M; ++i) {
            double s = 0.0;
            for (int j = 0; j < N; ++j) s += Kout[((size_t)k * M + i) * N + j] * zz[j];
            vk[i] = dout[(size_t)k * M + i] - s;
            v[(size_t)k * M + i] = vk[i];
        }
        double e[N];
        for (int i = 0; i < N; ++i) e[i] = ak[i] - zz[i];
        double c1 = 0.0;
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
            for (int j = 0; j < N; ++j) s += Qb[i][j] * e[j];
            c1 += e[i] * s;
        }
        double c2 = 0.0;
        for (int i = 0; i < M; ++i) {
            double s = 0.0;
            for (int j = 0; j < M; ++j) s += Rb[i][j] * vk[j];
            c2 += vk[i] * s;
        }
        cost += c1 + c2;
        double zn[N];
        for (int i = 0; i < N; ++i) {
            double s1 = 0.0;
            for (int j = 0; j < N; ++j) s1 += ((i == j ? 1.0 : 0.0) + dt * a[i * N + j]) * zz[j];
            double s2 = 0.0;
            for (int j = 0; j < M; ++j) s2 += (dt * b[i * M + j]) * vk[j];
            zn[i] = s1 + s2;
        }
        for (int i = 0; i < N; ++i) {
            zz[i] = zn[i];
            if (z) z[(size_t)(k + 1) * N + i] = zz[i];
        }
    }
    *cost_out = cost;
}

template <int N, int M>
__global__ void lqr_solve_kernel(int T, double dt, const double* A, const double* B,
                                 const double* Q, const double* R, const double* a, double* v,
                                 double* z, double* K, double* dff, double* scal, int* status) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    ArrayJac<N, M> jac{A, B};
    ArrayFlow<N> fl{a};
    double cost = 0.0;
    lqr_core<N, M>(jac, fl, T, dt, Q, R, K, dff, v, z, &cost, status);
    scal[0] = cost;
    scal[1] = 0.0;
}

template <class Mdl>
__global__ void plan_update_kernel(const double* prm, const double* S, const double* U, int T,
                                   double dt, int d, const double* P, const double* flow,
                                   const double* Q, const double* R, double eta,
                                   const double* clamp, double* Unext, double* lqr_costs,
                                   int* plan_state, int iteration, double* K, double* dff,
                                   double* v) {
    constexpr int N = Mdl::N, M = Mdl::M;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (plan_state && *((volatile int*)plan_state) != 0) return;
    ModelJac<Mdl> jac{prm, S, U};
    LiftedFlow<N> fl{flow, P, d};
    double cost = 0.0;
    int fail = -1;
    lqr_core<N, M>(jac, fl, T, dt, Q, R, K, dff, v, nullptr, &cost, &fail);
    if (fail >= 0) {
        plan_state[FCB_STATE_STOP] = 2;
        plan_state[FCB_STATE_STAGE] = 3;
        plan_state[FCB_STATE_ITER] = iteration;
        plan_state[FCB_STATE_INDEX] = fail;
        return;
    }
    lqr_costs[iteration] = cost;
    for (int k = 0; k < T; ++k)
        for (int j = 0; j < M; ++j) {
            double u = U[(size_t)k * M + j] + eta * v[(size_t)k * M + j];
            if (clamp) {
                const double b = clamp[j];
                u = fmin(fmax(u, -b), b);
            }
            Unext[(size_t)k * M + j] = u;
        }
    plan_state[FCB_STATE_UPDATES] = iteration + 1;
}

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

int rollout(int model, int ns, int m, const double* prm, const double* s0, const double* U, int T,
            double dt, double* S, int d, const double* P, double* X, int* status, int* plan_state,
            int iteration, cudaStream_t st) {
    int rc = check_dims(model, ns, m);
    if (rc) return rc;
    if (T < 1) return fail(FCB_EINPUT, "need at least one control step");
    FCB_MODEL_DISPATCH((rollout_kernel<Mdl><<<1, 32, 0, st>>>(prm, s0, U, T, dt, S, d, P, X, status,
                                                              plan_state, iteration)));
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

size_t lqr_ws_bytes(int ns, int m, int T) {
    return sizeof(double) * ((size_t)T * m * ns + (size_t)T * m + (size_t)T * m) + 256;
}

int lqr_solve(int ns, int m, int T, double dt, const double* A, const double* B, const double* Q,
              const double* R, const double* a, double* v, double* z, double* K, double* dff,
              double* scal, int* status, double* ws, cudaStream_t st) {
    if (T < 1) return fail(FCB_EINPUT, "horizon must be >= 1");
    double* Kb = K ? K : ws;
    double* db = dff ? dff : ws + (size_t)T * m * ns;
    if ((!K || !dff) && !ws) return fail(FCB_EWORKSPACE, "lqr needs a workspace for K/d");
#define FCB_LQR_CASE(NN, MM)                                                                     \
    case NN * 4 + MM:                                                                            \
        lqr_solve_kernel<NN, MM><<<1, 32, 0, st>>>(T, dt, A, B, Q, R, a, v, z, Kb, db, scal,      \
                                                   status);                                      \
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
    FCB_LAUNCHED("lqr_solve_kernel");
    return FCB_OK;
}

size_t plan_update_ws_bytes(int ns, int m, int T) {
    return sizeof(double) * ((size_t)T * m * ns + 2 * (size_t)T * m) + 512;
}

int plan_update(int model, int ns, int m, const double* prm, const double* S, const double* U,
                int T, double dt, int d, const double* P, const double* flow, const double* Q,
                const double* R, double eta, const double* clamp, double* Unext, double* lqr_costs,
                int* plan_state, int iteration, double* ws, size_t ws_bytes, cudaStream_t st) {
    int rc = check_dims(model, ns, m);
    if (rc) return rc;
    if (ws_bytes < plan_update_ws_bytes(ns, m, T))
        return fail(FCB_EWORKSPACE, "plan_update workspace too small");
    double* K = ws;
    double* dff = K + (size_t)T * m * ns;
    double* v = dff + (size_t)T * m;
    FCB_MODEL_DISPATCH((plan_update_kernel<Mdl><<<1, 32, 0, st>>>(
        prm, S, U, T, dt, d, P, flow, Q, R, eta, clamp, Unext, lqr_costs, plan_state, iteration, K,
        dff, v)));
    FCB_LAUNCHED("plan_update_kernel");
    return FCB_OK;
}

}  // namespace fcb
