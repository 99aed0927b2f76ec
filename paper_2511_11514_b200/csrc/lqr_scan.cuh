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

struct LqrScanArgs {
    int T;
    double dt;
    const double* Q;  // N x N (weights, not yet scaled by dt)
    const double* R;  // M x M
    double* agg;      // 2 * THREADS * ESZ   (suffix aggregates, ping-pong)
    double* aff;      // 2 * THREADS * (N*N+N)
    double* K;        // T * M * N
    double* dff;      // T * M
    double* v;        // T * M (may be null when U_next is given)
    double* z;        // (T+1) * N (nullable)
    double* cost;     // nullable device scalar
    int* fail;        // device int: -1 or the Riccati failure index
    // planner hooks (nullable)
    const double* U;
    double* U_next;
    double eta;
    const double* clamp;
    double* lqr_costs;
    int* plan_state;
    int iteration;
};

template <int N, int M, class Jac, class Flow>
__device__ void lqr_scan_body(const Jac& jac, const Flow& flow, const LqrScanArgs& p) {
    constexpr int ESZ = elem_doubles<N>();
    constexpr int ASZ = N * N + N;
    __shared__ double sQb[N][N], sRb[M][M], sRtinv[M][M];
    __shared__ int s_fail;
    __shared__ double s_red[32];
    const int tid = threadIdx.x;
    const int T = p.T;
    const double dt = p.dt;
    if (tid == 0) {
        s_fail = -1;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) sQb[i][j] = dt * p.Q[i * N + j];
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) sRb[i][j] = dt * p.R[i * M + j];
        // Rt^-1 = (2 Rb)^-1 by Gauss-Jordan on the tiny m x m matrix
        double Aa[M][2 * M];
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < 2 * M; ++j)
                Aa[i][j] = (j < M) ? 2.0 * sRb[i][j] : ((j - M == i) ? 1.0 : 0.0);
        for (int c = 0; c < M; ++c) {
            int pv = c;
            for (int r = c + 1; r < M; ++r)
                if (fabs(Aa[r][c]) > fabs(Aa[pv][c])) pv = r;
            for (int k = 0; k < 2 * M; ++k) {
                double t = Aa[c][k];
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
            for (int j = 0; j < M; ++j) sRtinv[i][j] = Aa[i][M + j];
    }
    __syncthreads();

    // elements 0..T (T is the zero terminal element)
    const int total = T + 1;
    const int L = (total + LQR_THREADS - 1) / LQR_THREADS;
    const int nch = (total + L - 1) / L;
    const int lo = tid * L, hi = min(lo + L, total);

    auto base_elem = [&](int k, Elem<N>& e) {
        if (k >= T) {
#pragma unroll
            for (int i = 0; i < N; ++i) {
                e.b[i] = 0.0;
                e.h[i] = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) e.A[i][j] = e.C[i][j] = e.J[i][j] = 0.0;
            }
            return;
        }
        double F[N][N], G[N][M], ak[N];
        step_data<N, M>(jac, flow, k, dt, F, G, ak);
        double GR[N][M];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) {
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < M; ++q) s += G[i][q] * sRtinv[q][j];
                GR[i][j] = s;
            }
#pragma unroll
        for (int i = 0; i < N; ++i) {
            e.b[i] = 0.0;
            double qa = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) qa += sQb[i][q] * ak[q];
            e.h[i] = 2.0 * qa;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                e.A[i][j] = F[i][j];
                e.J[i][j] = 2.0 * sQb[i][j];
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < M; ++q) s += GR[i][q] * G[j][q];
                e.C[i][j] = s;
            }
        }
    };

    // ---- P1: chunk aggregates (suffix products inside the chunk) ---------
    double* aggA = p.agg;
    double* aggB = p.agg + (size_t)LQR_THREADS * ESZ;
    if (tid < nch) {
        Elem<N> acc, e, tmp;
        base_elem(hi - 1, acc);
        for (int k = hi - 2; k >= lo; --k) {
            base_elem(k, e);
            elem_combine<N>(e, acc, tmp);
            acc = tmp;
        }
        elem_store<N>(aggA + (size_t)tid * ESZ, acc);
    }
    __syncthreads();
    // ---- P2: inclusive suffix scan over the aggregates (Hillis-Steele) ---
    double* src = aggA;
    double* dst = aggB;
    for (int s = 1; s < nch; s <<= 1) {
        if (tid < nch) {
            Elem<N> a, b, o;
            elem_load<N>(src + (size_t)tid * ESZ, a);
            if (tid + s < nch) {
                elem_load<N>(src + (size_t)(tid + s) * ESZ, b);
                elem_combine<N>(a, b, o);
                elem_store<N>(dst + (size_t)tid * ESZ, o);
            } else {
                elem_store<N>(dst + (size_t)tid * ESZ, a);
            }
        }
        __syncthreads();
        double* t = src;
        src = dst;
        dst = t;
    }
    // ---- P3: information-form re-walk, gains K_k, d_k --------------------
    if (tid < nch) {
        double J2[N][N], h2[N];
        if (tid + 1 < nch) {
            const double* sp = src + (size_t)(tid + 1) * ESZ;
#pragma unroll
            for (int i = 0; i < N * N; ++i) (&J2[0][0])[i] = __ldcg(sp + 2 * N * N + 2 * N + i);
#pragma unroll
            for (int i = 0; i < N; ++i) h2[i] = __ldcg(sp + 2 * N * N + N + i);
        } else {
#pragma unroll
            for (int i = 0; i < N; ++i) {
                h2[i] = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) J2[i][j] = 0.0;
            }
        }
        int local_fail = -1;
        for (int k = hi - 1; k >= lo; --k) {
            if (k < T) {
                // gains from the suffix k+1 (P' = J2/2, p' = -h2/2)
                double F[N][N], G[N][M], ak[N];
                step_data<N, M>(jac, flow, k, dt, F, G, ak);
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
                double H[M][M], rhs[M][N + 1];
#pragma unroll
                for (int i = 0; i < M; ++i) {
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        double s = 0.0;
#pragma unroll
                        for (int q = 0; q < N; ++q) s += G[q][i] * PG[q][j];
                        H[i][j] = sRb[i][j] + s;
                    }
#pragma unroll
                    for (int j = 0; j < N; ++j) {
                        double s = 0.0;
#pragma unroll
                        for (int q = 0; q < N; ++q) s += G[q][i] * PF[q][j];
                        rhs[i][j] = s;
                    }
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < N; ++q) s += G[q][i] * h2[q];
                    rhs[i][N] = 0.5 * s;  // -G' p' with p' = -h2/2
                }
                // H X = rhs (partial pivoting)
#pragma unroll
                for (int col = 0; col < M; ++col) {
                    int pv = col;
#pragma unroll
                    for (int r = col + 1; r < M; ++r)
                        if (fabs(H[r][col]) > fabs(H[pv][col])) pv = r;
                    if (pv != col) {
#pragma unroll
                        for (int q = 0; q < M; ++q) {
                            double t = H[col][q];
                            H[col][q] = H[pv][q];
                            H[pv][q] = t;
                        }
#pragma unroll
                        for (int q = 0; q < N + 1; ++q) {
                            double t = rhs[col][q];
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
                        for (int q = 0; q < N + 1; ++q) rhs[r][q] -= l * rhs[col][q];
                    }
                }
#pragma unroll
                for (int r = M - 1; r >= 0; --r)
#pragma unroll
                    for (int q = 0; q < N + 1; ++q) {
                        double vv = rhs[r][q];
#pragma unroll
                        for (int c2 = r + 1; c2 < M; ++c2) vv -= H[r][c2] * rhs[c2][q];
                        rhs[r][q] = vv / H[r][r];
                    }
#pragma unroll
                for (int i = 0; i < M; ++i) {
#pragma unroll
                    for (int j = 0; j < N; ++j) p.K[((size_t)k * M + i) * N + j] = rhs[i][j];
                    p.dff[(size_t)k * M + i] = rhs[i][N];
                }
                // advance the suffix to k (information form)
                Elem<N> e;
                base_elem(k, e);
                info_step<N>(e, J2, h2);
                bool finite = true;
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    finite = finite && isfinite(h2[i]);
#pragma unroll
                    for (int j = 0; j < N; ++j) finite = finite && isfinite(J2[i][j]);
                }
                if (!finite && local_fail < 0) local_fail = k;
            }
        }
        if (local_fail >= 0) atomicMax(&s_fail, local_fail);
    }
    __syncthreads();
    if (s_fail >= 0) {
        if (tid == 0) {
            *p.fail = s_fail;
            if (p.plan_state) {
                p.plan_state[FCB_STATE_STOP] = 2;
                p.plan_state[FCB_STATE_STAGE] = 3;
                p.plan_state[FCB_STATE_ITER] = p.iteration;
                p.plan_state[FCB_STATE_INDEX] = s_fail;
            }
        }
        return;
    }
    // ---- P4: chunk compositions of the closed-loop maps -------------------
    // maps for k = 0..T-1:  z_{k+1} = (F_k - G_k K_k) z_k + G_k d_k
    const int Lf = (T + LQR_THREADS - 1) / LQR_THREADS;
    const int nchf = (T + Lf - 1) / Lf;
    const int flo = tid * Lf, fhi = min(flo + Lf, T);
    auto step_map = [&](int k, Aff<N>& a) {
        double F[N][N], G[N][M], ak[N];
        step_data<N, M>(jac, flow, k, dt, F, G, ak);
        double Kk[M][N], dk[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
#pragma unroll
            for (int j = 0; j < N; ++j) Kk[i][j] = __ldcg(p.K + ((size_t)k * M + i) * N + j);
            dk[i] = __ldcg(p.dff + (size_t)k * M + i);
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double cc = 0.0;
#pragma unroll
            for (int q = 0; q < M; ++q) cc += G[i][q] * dk[q];
            a.c[i] = cc;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < M; ++q) s += G[i][q] * Kk[q][j];
                a.M[i][j] = F[i][j] - s;
            }
        }
    };
    double* affA = p.aff;
    double* affB = p.aff + (size_t)LQR_THREADS * ASZ;
    if (tid < nchf) {
        Aff<N> acc, m, tmp;
        aff_identity<N>(acc);
        for (int k = flo; k < fhi; ++k) {
            step_map(k, m);
            aff_compose<N>(m, acc, tmp);
            acc = tmp;
        }
        aff_store<N>(affA + (size_t)tid * ASZ, acc);
    }
    __syncthreads();
    // ---- P5: inclusive prefix scan over chunk maps ------------------------
    double* fs = affA;
    double* fd = affB;
    for (int s = 1; s < nchf; s <<= 1) {
        if (tid < nchf) {
            Aff<N> a, b, o;
            aff_load<N>(fs + (size_t)tid * ASZ, a);
            if (tid - s >= 0) {
                aff_load<N>(fs + (size_t)(tid - s) * ASZ, b);
                aff_compose<N>(a, b, o);
                aff_store<N>(fd + (size_t)tid * ASZ, o);
            } else {
                aff_store<N>(fd + (size_t)tid * ASZ, a);
            }
        }
        __syncthreads();
        double* t = fs;
        fs = fd;
        fd = t;
    }
    // ---- P6: re-walk: z, v*, cost, control update --------------------------
    double cost_part = 0.0;
    if (tid < nchf) {
        double zz[N];
        if (tid == 0) {
#pragma unroll
            for (int i = 0; i < N; ++i) zz[i] = 0.0;
        } else {  // z at chunk start = offset of the exclusive prefix (z_0 = 0)
#pragma unroll
            for (int i = 0; i < N; ++i) zz[i] = __ldcg(fs + (size_t)(tid - 1) * ASZ + N * N + i);
        }
        if (p.z && tid == 0)
#pragma unroll
            for (int i = 0; i < N; ++i) p.z[i] = 0.0;
        for (int k = flo; k < fhi; ++k) {
            double F[N][N], G[N][M], ak[N];
            step_data<N, M>(jac, flow, k, dt, F, G, ak);
            double vk[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) s += __ldcg(p.K + ((size_t)k * M + i) * N + j) * zz[j];
                vk[i] = __ldcg(p.dff + (size_t)k * M + i) - s;
            }
            double e[N];
#pragma unroll
            for (int i = 0; i < N; ++i) e[i] = ak[i] - zz[i];
            double c1 = 0.0, c2 = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) s += sQb[i][j] * e[j];
                c1 += e[i] * s;
            }
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < M; ++j) s += sRb[i][j] * vk[j];
                c2 += vk[i] * s;
            }
            cost_part += c1 + c2;
            if (p.v)
#pragma unroll
                for (int i = 0; i < M; ++i) p.v[(size_t)k * M + i] = vk[i];
            if (p.U_next) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    double u = p.U[(size_t)k * M + i] + p.eta * vk[i];
                    if (p.clamp) {
                        const double b = p.clamp[i];
                        u = fmin(fmax(u, -b), b);
                    }
                    p.U_next[(size_t)k * M + i] = u;
                }
            }
            double zn[N];
#pragma unroll
            for (int i = 0; i < N; ++i) {
                double s1 = 0.0, s2 = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) s1 += F[i][j] * zz[j];
#pragma unroll
                for (int j = 0; j < M; ++j) s2 += G[i][j] * vk[j];
                zn[i] = s1 + s2;
            }
#pragma unroll
            for (int i = 0; i < N; ++i) {
                zz[i] = zn[i];
                if (p.z) p.z[(size_t)(k + 1) * N + i] = zz[i];
            }
        }
    }
    const double total_cost = block_sum<LQR_THREADS>(cost_part, s_red);
    if (tid == 0) {
        *p.fail = -1;
        if (p.cost) *p.cost = total_cost;
        if (p.plan_state) {
            p.lqr_costs[p.iteration] = total_cost;
            p.plan_state[FCB_STATE_UPDATES] = p.iteration + 1;
        }
    }
}

}  // namespace fcb
