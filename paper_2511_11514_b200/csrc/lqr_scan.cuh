// lqr_scan.cuh -- parallel-in-time flow-matching LQR (one CTA per problem).
//
// Replaces the sequential backward Riccati / forward sweep of lqr.py:154-200
// by associative scans (temporal parallelisation of LQ control, Sarkka and
// Garcia-Fernandez): each time step k is an element
//     e_k = (A, b, C, eta, J) = (F_k, 0, G_k Rt^-1 G_k', 2 Qb a_k, 2 Qb),
// F = I + dt A_k, G = dt B_k, Rt = 2 dt R, with the combination
//     M   = (I + C1 J2)^-1
//     A   = A2 M A1            b = A2 M (b1 + C1 eta2) + b2
//     C   = A2 M C1 A2' + C2   eta = (M A1)' (eta2 - J2 b1) + eta1
//     J   = (M A1)' J2 A1 + J1
// The suffix product e_k (x) ... (x) e_T has J = 2 P_k and eta = -2 p_k of
// the reference's recursion, so the gains K_k, d_k of lqr.py:176-184 follow
// per step in parallel; the forward pass z_{k+1} = (F - G K) z + G d is an
// affine prefix scan.  Work O(T n^3), depth O(T/threads + log threads).
//
// Layout: THREADS chunks of L = ceil((T+1)/THREADS) consecutive steps.
//   P1 chunk aggregates (sequential combine inside a chunk)
//   P2 Hillis-Steele suffix scan over the aggregates (global, L2 resident)
//   P3 re-walk each chunk right-to-left in information form (J, eta only),
//      emitting K_k, d_k and the first non-finite index
//   P4 chunk compositions of the closed-loop affine maps
//   P5 Hillis-Steele prefix scan over them
//   P6 re-walk: z_k, v_k = d_k - K_k z_k, stage costs, optional U update
#pragma once

#include "fcb_internal.cuh"

namespace fcb {

constexpr int LQR_THREADS = 256;

template <int N>
struct Elem {
    double A[N][N];
    double b[N];
    double C[N][N];
    double h[N];
    double J[N][N];
};

template <int N>
__device__ __forceinline__ void elem_identity(Elem<N>& e) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        e.b[i] = 0.0;
        e.h[i] = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            e.A[i][j] = (i == j) ? 1.0 : 0.0;
            e.C[i][j] = 0.0;
            e.J[i][j] = 0.0;
        }
    }
}

// Solve (I + C1 J2) X = R for X (R: N x NR), partial pivoting.
template <int N, int NR>
__device__ __forceinline__ void solve_ipcj(const double (&C1)[N][N], const double (&J2)[N][N],
                                           double (&R)[N][NR]) {
    double Mt[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += C1[i][q] * J2[q][j];
            Mt[i][j] = s;
        }
#pragma unroll
    for (int col = 0; col < N; ++col) {
        int piv = col;
        double best = fabs(Mt[col][col]);
#pragma unroll
        for (int r = col + 1; r < N; ++r)
            if (fabs(Mt[r][col]) > best) {
                best = fabs(Mt[r][col]);
                piv = r;
            }
        if (piv != col) {
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const double t = Mt[col][k];
                Mt[col][k] = Mt[piv][k];
                Mt[piv][k] = t;
            }
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const double t = R[col][k];
                R[col][k] = R[piv][k];
                R[piv][k] = t;
            }
        }
        const double inv = 1.0 / Mt[col][col];
#pragma unroll
        for (int r = col + 1; r < N; ++r) {
            const double l = Mt[r][col] * inv;
#pragma unroll
            for (int k = col; k < N; ++k) Mt[r][k] -= l * Mt[col][k];
#pragma unroll
            for (int k = 0; k < NR; ++k) R[r][k] -= l * R[col][k];
        }
    }
#pragma unroll
    for (int r = N - 1; r >= 0; --r) {
        const double inv = 1.0 / Mt[r][r];
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            double v = R[r][k];
#pragma unroll
            for (int q = r + 1; q < N; ++q) v -= Mt[r][q] * R[q][k];
            R[r][k] = v * inv;
        }
    }
}

// out = e1 (x) e2   (e1 earlier in time).  out may alias neither input.
template <int N>
__device__ void elem_combine(const Elem<N>& e1, const Elem<N>& e2, Elem<N>& out) {
    // X = (I + C1 J2)^-1 [A1 | b1 + C1 h2 | C1]
    double X[N][2 * N + 1];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double ch = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) ch += e1.C[i][q] * e2.h[q];
#pragma unroll
        for (int j = 0; j < N; ++j) {
            X[i][j] = e1.A[i][j];
            X[i][N + 1 + j] = e1.C[i][j];
        }
        X[i][N] = e1.b[i] + ch;
    }
    solve_ipcj<N, 2 * N + 1>(e1.C, e2.J, X);
    // A = A2 XA ; b = A2 Xb + b2 ; T = A2 XC
    double T[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double a = 0.0, t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) {
                a += e2.A[i][q] * X[q][j];
                t += e2.A[i][q] * X[q][N + 1 + j];
            }
            out.A[i][j] = a;
            T[i][j] = t;
        }
        double bb = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) bb += e2.A[i][q] * X[q][N];
        out.b[i] = bb + e2.b[i];
    }
    // C = T A2' + C2 (symmetrised)
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double c = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) c += T[i][q] * e2.A[j][q];
            out.C[i][j] = c + e2.C[i][j];
        }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
            const double s = 0.5 * (out.C[i][j] + out.C[j][i]);
            out.C[i][j] = s;
            out.C[j][i] = s;
        }
    // h = XA' (h2 - J2 b1) + h1 ; J = XA' J2 A1 + J1 (symmetrised)
    double r[N], JA[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) s += e2.J[i][q] * e1.b[q];
        r[i] = e2.h[i] - s;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += e2.J[i][q] * e1.A[q][j];
            JA[i][j] = t;
        }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) s += X[q][i] * r[q];
        out.h[i] = s + e1.h[i];
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += X[q][i] * JA[q][j];
            out.J[i][j] = t + e1.J[i][j];
        }
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = i + 1; j < N; ++j) {
            const double s = 0.5 * (out.J[i][j] + out.J[j][i]);
            out.J[i][j] = s;
            out.J[j][i] = s;
        }
}

// Information-form step: (J, h) of e (x) (J2, h2), with e.b == 0.
template <int N>
__device__ __forceinline__ void info_step(const Elem<N>& e, double (&J2)[N][N], double (&h2)[N]) {
    double X[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) X[i][j] = e.A[i][j];
    solve_ipcj<N, N>(e.C, J2, X);
    double JA[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += J2[i][q] * e.A[q][j];
            JA[i][j] = t;
        }
    double Jn[N][N], hn[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) s += X[q][i] * h2[q];
        hn[i] = s + e.h[i];
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += X[q][i] * JA[q][j];
            Jn[i][j] = t + e.J[i][j];
        }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
        h2[i] = hn[i];
#pragma unroll
        for (int j = 0; j < N; ++j) J2[i][j] = 0.5 * (Jn[i][j] + Jn[j][i]);
    }
}

template <int N>
__device__ __forceinline__ void elem_load(const double* __restrict__ p, Elem<N>& e) {
    const double* src = p;
#pragma unroll
    for (int i = 0; i < N * N; ++i) (&e.A[0][0])[i] = __ldcg(src + i);
    src += N * N;
#pragma unroll
    for (int i = 0; i < N; ++i) e.b[i] = __ldcg(src + i);
    src += N;
#pragma unroll
    for (int i = 0; i < N * N; ++i) (&e.C[0][0])[i] = __ldcg(src + i);
    src += N * N;
#pragma unroll
    for (int i = 0; i < N; ++i) e.h[i] = __ldcg(src + i);
    src += N;
#pragma unroll
    for (int i = 0; i < N * N; ++i) (&e.J[0][0])[i] = __ldcg(src + i);
}

template <int N>
__device__ __forceinline__ void elem_store(double* __restrict__ p, const Elem<N>& e) {
    double* dst = p;
#pragma unroll
    for (int i = 0; i < N * N; ++i) dst[i] = (&e.A[0][0])[i];
    dst += N * N;
#pragma unroll
    for (int i = 0; i < N; ++i) dst[i] = e.b[i];
    dst += N;
#pragma unroll
    for (int i = 0; i < N * N; ++i) dst[i] = (&e.C[0][0])[i];
    dst += N * N;
#pragma unroll
    for (int i = 0; i < N; ++i) dst[i] = e.h[i];
    dst += N;
#pragma unroll
    for (int i = 0; i < N * N; ++i) dst[i] = (&e.J[0][0])[i];
}

template <int N>
constexpr int elem_doubles() {
    return 3 * N * N + 2 * N;
}

// affine map z -> M z + c
template <int N>
struct Aff {
    double M[N][N];
    double c[N];
};

template <int N>
__device__ __forceinline__ void aff_identity(Aff<N>& a) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        a.c[i] = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) a.M[i][j] = (i == j) ? 1.0 : 0.0;
    }
}

// out = later o earlier  (apply `earlier` first)
template <int N>
__device__ __forceinline__ void aff_compose(const Aff<N>& later, const Aff<N>& earlier, Aff<N>& out) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double cc = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) cc += later.M[i][q] * earlier.c[q];
        out.c[i] = cc + later.c[i];
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
__device__ __forceinline__ void aff_load(const double* p, Aff<N>& a) {
#pragma unroll
    for (int i = 0; i < N * N; ++i) (&a.M[0][0])[i] = __ldcg(p + i);
#pragma unroll
    for (int i = 0; i < N; ++i) a.c[i] = __ldcg(p + N * N + i);
}

template <int N>
__device__ __forceinline__ void aff_store(double* p, const Aff<N>& a) {
#pragma unroll
    for (int i = 0; i < N * N; ++i) p[i] = (&a.M[0][0])[i];
#pragma unroll
    for (int i = 0; i < N; ++i) p[N * N + i] = a.c[i];
}

// Everything a step needs: F = I + dt A_k, G = dt B_k, the state flow a_k.
template <int N, int M, class Jac, class Flow>
__device__ __forceinline__ void step_data(const Jac& jac, const Flow& flow, int k, double dt,
                                          double (&F)[N][N], double (&G)[N][M], double (&ak)[N]) {
    double a[N * N], b[N * M];
    jac.get(k, a, b);
    flow.get(k, ak);
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) F[i][j] = (i == j ? 1.0 : 0.0) + dt * a[i * N + j];
#pragma unroll
        for (int j = 0; j < M; ++j) G[i][j] = dt * b[i * M + j];
    }
}

}  // namespace fcb

#include "lqr_split.cuh"
