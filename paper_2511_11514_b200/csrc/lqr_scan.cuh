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
// Split in two phases: the Riccati phase (lqr_split.cuh, one CTA) emits the
// per-step K, H^-1 G', Phi, Acl, G; the affine phase (eta backward, z forward)
// runs as affine scans (affscan.cuh, plan_scan.cuh).  This header holds the
// shared (I + C J)^-1 solve.
#pragma once

#include "fcb_internal.cuh"

namespace fcb {

constexpr int LQR_THREADS = 256;

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
}  // namespace fcb

#include "lqr_split.cuh"
