// lqr_split.cuh -- the parallel-in-time LQR split into a Riccati phase and an
// affine phase.
//
// In the element e_k = (A, b, C, eta, J) = (F_k, 0, G Rt^-1 G', 2 Qb a_k, 2 Qb)
// only eta depends on the flow a_k.  The (A, C, J) parts, the value matrices
// J_k = 2 P_k, the gains K_k = H^-1 G' P' F, the maps H^-1 G' and the
// closed-loop matrices depend on the linearisation alone:
//
//   Riccati phase  (flow-independent; a suffix scan of (A, C, J) elements)
//     emits  K_k, L_k = H_k^-1 G_k', Phi_k = (I + C_k J_{k+1})^-1 F_k,
//            Acl_k = F_k - G_k K_k, G_k
//   affine phase   (per flow; two O(T n^2)-work affine scans)
//     eta_k = Phi_k' eta_{k+1} + 2 Qb a_k   (eta_T = 0; eta = -2 p)
//     d_k   = 1/2 L_k eta_{k+1}             (lqr.py:182-184)
//     z_{k+1} = Acl_k z_k + G_k d_k, v_k = d_k - K_k z_k, cost, U update
//
// For models whose Jacobians do not depend on the state (single/double
// integrator, LTI) the Riccati-phase inputs are bitwise identical in every
// outer iteration of plan(), so the planner runs it once per plan() call and
// only the affine phase per iteration.  Nonlinear models run both phases every
// iteration.
#pragma once

#include "fcb_internal.cuh"

namespace fcb {

template <int N>
struct ElemR {
    double A[N][N];
    double C[N][N];
    double J[N][N];
};

template <int N>
constexpr int elemr_doubles() {
    return 3 * N * N;
}

// out = e1 (x) e2 on the (A, C, J) parts.  out aliases neither input.
template <int N>
__device__ void elemr_combine(const ElemR<N>& e1, const ElemR<N>& e2, ElemR<N>& out) {
    double X[N][2 * N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            X[i][j] = e1.A[i][j];
            X[i][N + j] = e1.C[i][j];
        }
    solve_ipcj<N, 2 * N>(e1.C, e2.J, X);
    double T[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double a = 0.0, t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) {
                a += e2.A[i][q] * X[q][j];
                t += e2.A[i][q] * X[q][N + j];
            }
            out.A[i][j] = a;
            T[i][j] = t;
        }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double c = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) c += T[i][q] * e2.A[j][q];
            out.C[i][j] = c + e2.C[i][j];
        }
    double JA[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += e2.J[i][q] * e1.A[q][j];
            JA[i][j] = t;
        }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += X[q][i] * JA[q][j];
            out.J[i][j] = t + e1.J[i][j];
        }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
            const double c = 0.5 * (out.C[i][j] + out.C[j][i]);
            out.C[i][j] = c;
            out.C[j][i] = c;
            const double s = 0.5 * (out.J[i][j] + out.J[j][i]);
            out.J[i][j] = s;
            out.J[j][i] = s;
        }
}

template <int N>
__device__ __forceinline__ void elemr_load(const double* __restrict__ p, ElemR<N>& e) {
#pragma unroll
    for (int i = 0; i < N * N; ++i) {
        (&e.A[0][0])[i] = __ldcg(p + i);
        (&e.C[0][0])[i] = __ldcg(p + N * N + i);
        (&e.J[0][0])[i] = __ldcg(p + 2 * N * N + i);
    }
}

template <int N>
__device__ __forceinline__ void elemr_store(double* __restrict__ p, const ElemR<N>& e) {
#pragma unroll
    for (int i = 0; i < N * N; ++i) {
        p[i] = (&e.A[0][0])[i];
        p[N * N + i] = (&e.C[0][0])[i];
        p[2 * N * N + i] = (&e.J[0][0])[i];
    }
}

template <int N, int M>
struct LqrShared {
    double Qb[N][N], Rb[M][M], Rtinv[M][M];
    int fail;
    double red[32];
};

template <int N, int M>
__device__ void lqr_shared_init(LqrShared<N, M>& s, const double* Q, const double* R, double dt) {
    if (threadIdx.x == 0) {
        s.fail = -1;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) s.Qb[i][j] = dt * Q[i * N + j];
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) s.Rb[i][j] = dt * R[i * M + j];
        // Rt^-1 = (2 Rb)^-1, Gauss-Jordan with partial pivoting (m <= 3)
        double Aa[M][2 * M];
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < 2 * M; ++j)
                Aa[i][j] = (j < M) ? 2.0 * s.Rb[i][j] : ((j - M == i) ? 1.0 : 0.0);
        for (int c = 0; c < M; ++c) {
            int pv = c;
            for (int r = c + 1; r < M; ++r)
                if (fabs(Aa[r][c]) > fabs(Aa[pv][c])) pv = r;
            for (int k = 0; k < 2 * M; ++k) {
                const double t = Aa[c][k];
                Aa[c][k] = Aa[pv][k];
                Aa[pv][k] = t;
            }
            const double inv = 1.0 / Aa[c][c];
            for (int k = 0; k < 2 * M; ++k) Aa[c][k] *= inv;
            for (int r = 0; r < M; ++r)
                if (r != c) {
                    const double l = Aa[r][c];
                    for (int k = 0; k < 2 * M; ++k) Aa[r][k] -= l * Aa[c][k];
                }
        }
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) s.Rtinv[i][j] = Aa[i][M + j];
    }
    __syncthreads();
}

struct RicArgs {
    int T;
    double dt;
    const double* Q;
    const double* R;
    double* agg;  // 2 * LQR_THREADS * 3N^2
    // per-step outputs, element-major: X[e * T + k]
    double* K;    // M*N x T
    double* Lg;   // M*N x T   H^-1 G'
    double* Acl;  // N*N x T   closed loop F - G K
    double* Gm;   // N*M x T
    int* fail;
    int* plan_state;
    int iteration;
};

// Riccati phase: suffix scan of (A, C, J), then per step the gains.
template <int N, int M, class Jac>
__device__ void riccati_body(const Jac& jac, const RicArgs& p) {
    constexpr int ESZ = elemr_doubles<N>();
    __shared__ LqrShared<N, M> sh;
    lqr_shared_init<N, M>(sh, p.Q, p.R, p.dt);
    const int tid = threadIdx.x;
    const int T = p.T;
    const double dt = p.dt;
    const int total = T + 1;  // element T is the zero terminal element
    const int L = (total + LQR_THREADS - 1) / LQR_THREADS;
    const int nch = (total + L - 1) / L;
    const int lo = tid * L, hi = min(lo + L, total);

    auto fg = [&](int k, double (&F)[N][N], double (&G)[N][M]) {
        double a[N * N], b[N * M];
        jac.get(k, a, b);
#pragma unroll
        for (int i = 0; i < N; ++i) {
#pragma unroll
            for (int j = 0; j < N; ++j) F[i][j] = (i == j ? 1.0 : 0.0) + dt * a[i * N + j];
#pragma unroll
            for (int j = 0; j < M; ++j) G[i][j] = dt * b[i * M + j];
        }
    };
    auto base = [&](int k, ElemR<N>& e) {
        if (k >= T) {
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) e.A[i][j] = e.C[i][j] = e.J[i][j] = 0.0;
            return;
        }
        double F[N][N], G[N][M];
        fg(k, F, G);
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) {
                e.A[i][j] = F[i][j];
                e.J[i][j] = 2.0 * sh.Qb[i][j];
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < M; ++q) {
                    double gr = 0.0;
#pragma unroll
                    for (int r = 0; r < M; ++r) gr += G[i][r] * sh.Rtinv[r][q];
                    s += gr * G[j][q];
                }
                e.C[i][j] = s;
            }
    };

    double* src = p.agg;
    double* dst = p.agg + (size_t)LQR_THREADS * ESZ;
    if (tid < nch) {  // P1: chunk aggregates
        ElemR<N> acc, e, tmp;
        base(hi - 1, acc);
        for (int k = hi - 2; k >= lo; --k) {
            base(k, e);
            elemr_combine<N>(e, acc, tmp);
            acc = tmp;
        }
        elemr_store<N>(src + (size_t)tid * ESZ, acc);
    }
    __syncthreads();
    for (int s = 1; s < nch; s <<= 1) {  // P2: inclusive suffix scan
        if (tid < nch) {
            ElemR<N> a, b, o;
            elemr_load<N>(src + (size_t)tid * ESZ, a);
            if (tid + s < nch) {
                elemr_load<N>(src + (size_t)(tid + s) * ESZ, b);
                elemr_combine<N>(a, b, o);
                elemr_store<N>(dst + (size_t)tid * ESZ, o);
            } else {
                elemr_store<N>(dst + (size_t)tid * ESZ, a);
            }
        }
        __syncthreads();
        double* t = src;
        src = dst;
        dst = t;
    }
    if (tid < nch) {  // P3: information-form re-walk, gains
        double J2[N][N];
        if (tid + 1 < nch) {
            const double* sp = src + (size_t)(tid + 1) * ESZ + 2 * N * N;
#pragma unroll
            for (int i = 0; i < N * N; ++i) (&J2[0][0])[i] = __ldcg(sp + i);
        } else {
#pragma unroll
            for (int i = 0; i < N * N; ++i) (&J2[0][0])[i] = 0.0;
        }
        int local_fail = -1;
        for (int k = hi - 1; k >= lo; --k) {
            if (k >= T) continue;
            double F[N][N], G[N][M];
            fg(k, F, G);
            // H = Rb + G' P' G, [K | Lg] = H^-1 [G' P' F | G'],  P' = J2 / 2
            double PG[N][M], PF[N][N];
#pragma unroll
            for (int i = 0; i < N; ++i) {
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < N; ++q) s += J2[i][q] * G[q][j];
                    PG[i][j] = 0.5 * s;
                }
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < N; ++q) s += J2[i][q] * F[q][j];
                    PF[i][j] = 0.5 * s;
                }
            }
            double H[M][M], rhs[M][2 * N];
#pragma unroll
            for (int i = 0; i < M; ++i) {
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < N; ++q) s += G[q][i] * PG[q][j];
                    H[i][j] = sh.Rb[i][j] + s;
                }
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < N; ++q) s += G[q][i] * PF[q][j];
                    rhs[i][j] = s;
                    rhs[i][N + j] = G[j][i];
                }
            }
#pragma unroll
            for (int col = 0; col < M; ++col) {  // Gaussian elimination, partial pivoting
                int pv = col;
#pragma unroll
                for (int r = col + 1; r < M; ++r)
                    if (fabs(H[r][col]) > fabs(H[pv][col])) pv = r;
                if (pv != col) {
#pragma unroll
                    for (int q = 0; q < M; ++q) {
                        const double t = H[col][q];
                        H[col][q] = H[pv][q];
                        H[pv][q] = t;
                    }
#pragma unroll
                    for (int q = 0; q < 2 * N; ++q) {
                        const double t = rhs[col][q];
                        rhs[col][q] = rhs[pv][q];
                        rhs[pv][q] = t;
                    }
                }
#pragma unroll
                for (int r = col + 1; r < M; ++r) {
                    const double l = H[r][col] / H[col][col];
#pragma unroll
                    for (int q = col; q < M; ++q) H[r][q] -= l * H[col][q];
#pragma unroll
                    for (int q = 0; q < 2 * N; ++q) rhs[r][q] -= l * rhs[col][q];
                }
            }
#pragma unroll
            for (int r = M - 1; r >= 0; --r)
#pragma unroll
                for (int q = 0; q < 2 * N; ++q) {
                    double v = rhs[r][q];
#pragma unroll
                    for (int c2 = r + 1; c2 < M; ++c2) v -= H[r][c2] * rhs[c2][q];
                    rhs[r][q] = v / H[r][r];
                }
            // per-step outputs, element-major ([element][T]): the affine scans
            // read one element of consecutive steps per warp load
            const size_t TT = (size_t)p.T;
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    p.K[(i * N + j) * TT + k] = rhs[i][j];
                    p.Lg[(i * N + j) * TT + k] = rhs[i][N + j];
                }
#pragma unroll
            for (int i = 0; i < N; ++i) {
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < M; ++q) s += G[i][q] * rhs[q][j];
                    p.Acl[(i * N + j) * TT + k] = F[i][j] - s;
                }
#pragma unroll
                for (int j = 0; j < M; ++j) p.Gm[(i * M + j) * TT + k] = G[i][j];
            }
            // Phi = (I + C_k J2)^-1 F ; J_k = Phi' J2 F + 2 Qb
            ElemR<N> e;
            base(k, e);
            double X[N][N];
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) X[i][j] = F[i][j];
            solve_ipcj<N, N>(e.C, J2, X);
            double JF[N][N], Jn[N][N];
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < N; ++q) s += J2[i][q] * F[q][j];
                    JF[i][j] = s;
                }
            bool finite = true;
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < N; ++q) s += X[q][i] * JF[q][j];
                    Jn[i][j] = s + 2.0 * sh.Qb[i][j];
                }
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) {
                    J2[i][j] = 0.5 * (Jn[i][j] + Jn[j][i]);
                    finite = finite && isfinite(J2[i][j]);
                }
            if (!finite && local_fail < 0) local_fail = k;
        }
        if (local_fail >= 0) atomicMax(&sh.fail, local_fail);
    }
    __syncthreads();
    if (tid == 0) {
        *p.fail = sh.fail;
        if (sh.fail >= 0 && p.plan_state) {
            p.plan_state[FCB_STATE_STOP] = 2;
            p.plan_state[FCB_STATE_STAGE] = 3;
            p.plan_state[FCB_STATE_ITER] = p.iteration;
            p.plan_state[FCB_STATE_INDEX] = sh.fail;
        }
    }
}

}  // namespace fcb
