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

#include <algorithm>

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

// ---------------------------------------------------------------------------
// Riccati phase over the whole GPU, warp-cooperative.
//
// The (A, C, J) element of a 6-state model is 108 doubles; a thread-private
// combine needs three of them live and spills to local memory, which at
// 10^5 steps turns the scan into an HBM-bound local-memory stream.  Here one
// WARP owns a chunk of consecutive elements and every element operation is
// spread over its 32 lanes, with the operands in the warp's shared-memory
// slice:
//   K1  each warp folds its chunk into one aggregate (suffix order); the CTA
//       runs a Hillis-Steele suffix scan over its warps' aggregates;
//   K2  one CTA scans the CTA aggregates;
//   K3  each warp forms J after its chunk (next warp's in-CTA suffix composed
//       with the next CTAs' suffix) and re-walks the chunk in information form,
//       emitting K_k, H_k^-1 G_k', Acl_k, G_k per step.
// ---------------------------------------------------------------------------
constexpr int RW_WARPS = 32;              // warps per CTA (K1, K3)
constexpr int RW_BLOCK = 32 * RW_WARPS;
constexpr int RW_K2_WARPS = 32;
constexpr int RW_MIN_CHUNK = 8;
#ifndef FCB_RIC_GENERIC
#define FCB_RIC_GENERIC 0  // 1: generic (A, C, J) combines in the K1 walk and the K3 Phi solve
#endif

struct RicArgs {
    int T;
    double dt;
    const double* Q;
    const double* R;
    int L;        // elements per warp chunk
    int nwarp;    // warps with a chunk slot (nblk * RW_WARPS)
    int nblk;     // CTAs of K1 / K3
    double* agg;  // 2 * nwarp * 3N^2: warp aggregates -> in-CTA suffixes (ping-pong)
    double* bagg; // (2 nblk + 2 RW_K2_WARPS) * 3N^2: CTA aggregates, their suffix scan, K2 scratch
    // per-step outputs, element-major: X[e * T + k]
    double* K;    // M*N x T
    double* Lg;   // M*N x T   H^-1 G'
    double* Acl;  // N*N x T   closed loop F - G K
    double* Gm;   // N*M x T
    int* fail;
    int* plan_state;
    int iteration;
};

// Number of Hillis-Steele rounds over `n` items (the result sits in buffer
// rounds & 1 of a ping-pong pair).
__host__ __device__ __forceinline__ int hs_rounds(int n) {
    int r = 0;
    for (int s = 1; s < n; s <<= 1) ++r;
    return r;
}

// Shared-memory slice of one warp.
template <int N, int M>
struct RwWarp {
    double E[3][3 * N * N];  // element slots (A | C | J, row-major)
    double Mt[N * N];
    double W[N * 2 * N];
    double Tm[N * N];
    double JA[N * N];
    double F[N * N];
    double G[N * M];
    double J2[N * N];
    double PG[N * M];
    double H[M * M];
    double rhs[M * 2 * N];
};

template <int N, int M>
constexpr size_t rw_smem_bytes(int warps) {
    return sizeof(LqrShared<N, M>) + (size_t)warps * sizeof(RwWarp<N, M>);
}

// In-place Gauss-Jordan elimination with partial pivoting by one warp:
// Mt (n x n) X = W (n x r); on return W holds X.  n <= 6, r <= 12.
template <int NN, int RR>
__device__ __forceinline__ void warp_gauss_jordan(double* Mt, double* W, int lane) {
    constexpr int C = NN + RR;
    constexpr int TOT = NN * C;
    constexpr int PER = (TOT + 31) / 32;
    for (int col = 0; col < NN; ++col) {
        int piv = col;
        double best = fabs(Mt[col * NN + col]);
        for (int r = col + 1; r < NN; ++r) {
            const double v = fabs(Mt[r * NN + col]);
            if (v > best) {
                best = v;
                piv = r;
            }
        }
        if (piv != col) {
            for (int c = lane; c < C; c += 32) {
                double* a = c < NN ? &Mt[col * NN + c] : &W[col * RR + c - NN];
                double* b = c < NN ? &Mt[piv * NN + c] : &W[piv * RR + c - NN];
                const double t = *a;
                *a = *b;
                *b = t;
            }
            __syncwarp();
        }
        const double inv = 1.0 / Mt[col * NN + col];
        double v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int idx = lane + 32 * k;
            if (idx < TOT) {
                const int r = idx / C, c = idx % C;
                const double pr = (c < NN ? Mt[col * NN + c] : W[col * RR + c - NN]) * inv;
                const double cur = c < NN ? Mt[r * NN + c] : W[r * RR + c - NN];
                v[k] = (r == col) ? pr : cur - Mt[r * NN + col] * pr;
            }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int idx = lane + 32 * k;
            if (idx < TOT) {
                const int r = idx / C, c = idx % C;
                if (c < NN) Mt[r * NN + c] = v[k];
                else W[r * RR + c - NN] = v[k];
            }
        }
        __syncwarp();
    }
}

// out = e1 (x) e2 (e1 earlier in time) on (A, C, J), by one warp:
//   X = (I + C1 J2)^-1 [A1 | C1],  A = A2 X_A,  C = A2 X_C A2' + C2,
//   J = X_A' J2 A1 + J1  (then C, J symmetrised).
template <int N, int M>
__device__ void warp_combine(const double* e1, const double* e2, double* out, RwWarp<N, M>& w,
                             int lane) {
    constexpr int NN = N * N;
    const double *A1 = e1, *C1 = e1 + NN, *J1 = e1 + 2 * NN;
    const double *A2 = e2, *C2 = e2 + NN, *J2 = e2 + 2 * NN;
    double *oA = out, *oC = out + NN, *oJ = out + 2 * NN;
    for (int idx = lane; idx < NN; idx += 32) {
        const int i = idx / N, j = idx % N;
        double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) s += C1[i * N + q] * J2[q * N + j];
        w.Mt[idx] = s;
    }
    for (int idx = lane; idx < 2 * NN; idx += 32) {
        const int i = idx / (2 * N), j = idx % (2 * N);
        w.W[idx] = j < N ? A1[i * N + j] : C1[i * N + j - N];
    }
    __syncwarp();
    warp_gauss_jordan<N, 2 * N>(w.Mt, w.W, lane);
    for (int idx = lane; idx < 2 * NN; idx += 32) {
        const int i = idx / (2 * N), j = idx % (2 * N);
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) s += A2[i * N + q] * w.W[q * 2 * N + j];
        if (j < N) oA[i * N + j] = s;
        else w.Tm[i * N + j - N] = s;
    }
    for (int idx = lane; idx < NN; idx += 32) {
        const int i = idx / N, j = idx % N;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) s += J2[i * N + q] * A1[q * N + j];
        w.JA[idx] = s;
    }
    __syncwarp();
    for (int idx = lane; idx < NN; idx += 32) {
        const int i = idx / N, j = idx % N;
        double c = 0.0, t = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            c += w.Tm[i * N + q] * A2[j * N + q];
            t += w.W[q * 2 * N + i] * w.JA[q * N + j];
        }
        oC[idx] = c + C2[idx];
        oJ[idx] = t + J1[idx];
    }
    __syncwarp();
    for (int idx = lane; idx < NN; idx += 32) {
        const int i = idx / N, j = idx % N;
        if (i < j) {
            const double c = 0.5 * (oC[i * N + j] + oC[j * N + i]);
            const double t = 0.5 * (oJ[i * N + j] + oJ[j * N + i]);
            oC[i * N + j] = c;
            oC[j * N + i] = c;
            oJ[i * N + j] = t;
            oJ[j * N + i] = t;
        }
    }
    __syncwarp();
}

// F = I + dt A_k, G = dt B_k into the warp slice (lane 0 evaluates the model).
template <int N, int M, class Jac>
__device__ __forceinline__ void warp_fg(const Jac& jac, int k, double dt, RwWarp<N, M>& w,
                                        int lane) {
    if (lane == 0) {
        double a[N * N], b[N * M];
        jac.get(k, a, b);
#pragma unroll
        for (int i = 0; i < N; ++i) {
#pragma unroll
            for (int j = 0; j < N; ++j) w.F[i * N + j] = (i == j ? 1.0 : 0.0) + dt * a[i * N + j];
#pragma unroll
            for (int j = 0; j < M; ++j) w.G[i * M + j] = dt * b[i * M + j];
        }
    }
    __syncwarp();
}

// Base element e_k = (F, G Rt^-1 G', 2 Qb) from the slice's F, G; zero for
// the terminal element.
template <int N, int M>
__device__ __forceinline__ void warp_base(bool terminal, const LqrShared<N, M>& sh, double* e,
                                          RwWarp<N, M>& w, int lane) {
    constexpr int NN = N * N;
    for (int idx = lane; idx < NN; idx += 32) {
        const int i = idx / N, j = idx % N;
        if (terminal) {
            e[idx] = e[NN + idx] = e[2 * NN + idx] = 0.0;
            continue;
        }
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) {
            double gr = 0.0;
#pragma unroll
            for (int r = 0; r < M; ++r) gr += w.G[i * M + r] * sh.Rtinv[r][q];
            s += gr * w.G[j * M + q];
        }
        e[idx] = w.F[idx];
        e[NN + idx] = s;
        e[2 * NN + idx] = 2.0 * sh.Qb[i][j];
    }
    __syncwarp();
}

// out = e_k (x) acc for the step-k base element e_k = (F, G Rt^-1 G', 2 Qb)
// of the slice's F, G (the chunk walk of K1).  With C_k of rank M the 6 x 6
// solve of the generic combine collapses (Woodbury, Rt = 2 Rb):
//   (I + C_k J2)^-1 = I - G (2H)^-1 G' J2,   H = Rb + G' (J2/2) G   (M x M)
//   X_A = F - G K = Acl,  K = H^-1 G' (J2/2) F;   X_C = 1/2 G H^-1 G'
// so  A = A2 Acl,  C = 1/2 (A2 G) H^-1 (A2 G)' + C2,  J = Acl' J2 F + 2 Qb
// -- the Riccati step itself, one M x M solve instead of an N x N one.
template <int N, int M>
__device__ void warp_combine_base(const double* acc, double* out, const LqrShared<N, M>& sh,
                                  RwWarp<N, M>& w, int lane) {
    constexpr int NN = N * N;
    const double *A2 = acc, *C2 = acc + NN, *J2 = acc + 2 * NN;
    double *oA = out, *oC = out + NN, *oJ = out + 2 * NN;
    // PG = (J2/2) G, AG = A2 G (N x M, AG in Tm), JF = J2 F (N x N, in JA)
    for (int idx = lane; idx < 2 * N * M + NN; idx += 32) {
        if (idx < 2 * N * M) {
            const int which = idx / (N * M), e = idx % (N * M), i = e / M, j = e % M;
            const double* L = which ? A2 : J2;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += L[i * N + q] * w.G[q * M + j];
            if (which) w.Tm[e] = s;
            else w.PG[e] = 0.5 * s;
        } else {
            const int e = idx - 2 * N * M, i = e / N, j = e % N;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += J2[i * N + q] * w.F[q * N + j];
            w.JA[e] = s;
        }
    }
    __syncwarp();
    // H = Rb + G' PG;  rhs = [G' JF / 2 | (A2 G)']
    for (int idx = lane; idx < M * M + M * 2 * N; idx += 32) {
        if (idx < M * M) {
            const int i = idx / M, j = idx % M;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += w.G[q * M + i] * w.PG[q * M + j];
            w.H[idx] = sh.Rb[i][j] + s;
        } else {
            const int e = idx - M * M, i = e / (2 * N), j = e % (2 * N);
            double s;
            if (j < N) {
                s = 0.0;
#pragma unroll
                for (int q = 0; q < N; ++q) s += w.G[q * M + i] * w.JA[q * N + j];
                s *= 0.5;
            } else {
                s = w.Tm[(j - N) * M + i];
            }
            w.rhs[e] = s;
        }
    }
    __syncwarp();
    warp_gauss_jordan<M, 2 * N>(w.H, w.rhs, lane);  // rhs <- [K | H^-1 (A2 G)']
    // Acl = F - G K (in Mt);  C = 1/2 (A2 G) H^-1 (A2 G)' + C2
    for (int idx = lane; idx < NN; idx += 32) {
        const int i = idx / N, j = idx % N;
        double a = 0.0, c = 0.0;
#pragma unroll
        for (int q = 0; q < M; ++q) {
            a += w.G[i * M + q] * w.rhs[q * 2 * N + j];
            c += w.Tm[i * M + q] * w.rhs[q * 2 * N + N + j];
        }
        w.Mt[idx] = w.F[idx] - a;
        oC[idx] = 0.5 * c + C2[idx];
    }
    __syncwarp();
    // A = A2 Acl;  J = Acl' JF + 2 Qb
    for (int idx = lane; idx < NN; idx += 32) {
        const int i = idx / N, j = idx % N;
        double a = 0.0, t = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            a += A2[i * N + q] * w.Mt[q * N + j];
            t += w.Mt[q * N + i] * w.JA[q * N + j];
        }
        oA[idx] = a;
        oJ[idx] = t + 2.0 * sh.Qb[i][j];
    }
    __syncwarp();
    for (int idx = lane; idx < NN; idx += 32) {
        const int i = idx / N, j = idx % N;
        if (i < j) {
            const double c = 0.5 * (oC[i * N + j] + oC[j * N + i]);
            const double t = 0.5 * (oJ[i * N + j] + oJ[j * N + i]);
            oC[i * N + j] = c;
            oC[j * N + i] = c;
            oJ[i * N + j] = t;
            oJ[j * N + i] = t;
        }
    }
    __syncwarp();
}

template <int N>
__device__ __forceinline__ void warp_identity(double* e, int lane) {
    constexpr int NN = N * N;
    for (int idx = lane; idx < NN; idx += 32) {
        e[idx] = (idx / N == idx % N) ? 1.0 : 0.0;
        e[NN + idx] = 0.0;
        e[2 * NN + idx] = 0.0;
    }
    __syncwarp();
}

template <int N>
__device__ __forceinline__ void warp_copy(const double* src, double* dst, int lane) {
    for (int idx = lane; idx < 3 * N * N; idx += 32) dst[idx] = __ldcg(src + idx);
    __syncwarp();
}

template <int N>
__device__ __forceinline__ void warp_store(const double* src, double* dst, int lane) {
    for (int idx = lane; idx < 3 * N * N; idx += 32) dst[idx] = src[idx];
    __syncwarp();
}

// K1: chunk aggregates + in-CTA suffix scan over warps.
template <int N, int M, class Jac>
__device__ void riccati_k1(const Jac& jac, const RicArgs& p) {
    constexpr int ESZ = elemr_doubles<N>();
    extern __shared__ __align__(16) unsigned char rw_smem[];
    LqrShared<N, M>& sh = *reinterpret_cast<LqrShared<N, M>*>(rw_smem);
    RwWarp<N, M>* slices = reinterpret_cast<RwWarp<N, M>*>(rw_smem + sizeof(LqrShared<N, M>));
    lqr_shared_init<N, M>(sh, p.Q, p.R, p.dt);
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    RwWarp<N, M>& w = slices[wl];
    const int gw = blockIdx.x * RW_WARPS + wl;
    const int total = p.T + 1;
    const int lo = gw * p.L, hi = min(lo + p.L, total);
    if (gw == 0 && lane == 0) *p.fail = -1;
    double* acc = w.E[0];
    double* e = w.E[1];
    double* out = w.E[2];
    if (lo < total) {
        const int k0 = hi - 1;
        if (k0 < p.T) warp_fg<N, M>(jac, k0, p.dt, w, lane);
        warp_base<N, M>(k0 >= p.T, sh, acc, w, lane);
        for (int k = hi - 2; k >= lo; --k) {
            warp_fg<N, M>(jac, k, p.dt, w, lane);  // k < T here
#if FCB_RIC_GENERIC
            warp_base<N, M>(false, sh, e, w, lane);
            warp_combine<N, M>(e, acc, out, w, lane);
#else
            warp_combine_base<N, M>(acc, out, sh, w, lane);
#endif
            double* t = acc;
            acc = out;
            out = t;
        }
    } else {
        warp_identity<N>(acc, lane);
    }
    double* src = p.agg;
    double* dst = p.agg + (size_t)p.nwarp * ESZ;
    warp_store<N>(acc, src + (size_t)gw * ESZ, lane);
    __syncthreads();
    for (int s = 1; s < RW_WARPS; s <<= 1) {
        if (wl + s < RW_WARPS) {
            warp_copy<N>(src + (size_t)(gw + s) * ESZ, e, lane);
            warp_combine<N, M>(acc, e, out, w, lane);
            double* t = acc;
            acc = out;
            out = t;
        }
        warp_store<N>(acc, dst + (size_t)gw * ESZ, lane);
        __syncthreads();
        double* t = src;
        src = dst;
        dst = t;
    }
    if (wl == 0) warp_store<N>(acc, p.bagg + (size_t)blockIdx.x * ESZ, lane);
}

// K2 (one CTA of RW_K2_WARPS warps): inclusive suffix scan over the CTA
// aggregates (bagg slot 0) into bagg slot 1, in three phases so each warp runs
// ~3 sqrt(nblk)-ish combines instead of log2(nblk) rounds of several:
//   1. warp w folds its contiguous group of aggregates into local suffixes;
//   2. Hillis-Steele suffix scan over the (<= 32) group aggregates;
//   3. every local suffix is completed with the suffix of the next groups.
template <int N, int M>
__device__ void riccati_k2(const RicArgs& p) {
    constexpr int ESZ = elemr_doubles<N>();
    extern __shared__ __align__(16) unsigned char rw_smem[];
    RwWarp<N, M>* slices = reinterpret_cast<RwWarp<N, M>*>(rw_smem + sizeof(LqrShared<N, M>));
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    RwWarp<N, M>& w = slices[wl];
    const int nb = p.nblk;
    const double* agg = p.bagg;
    double* suf = p.bagg + (size_t)nb * ESZ;
    double* gbuf = p.bagg + (size_t)2 * nb * ESZ;  // 2 x RW_K2_WARPS group slots
    const int G = (nb + RW_K2_WARPS - 1) / RW_K2_WARPS;
    const int ng = (nb + G - 1) / G;
    const int lo = wl * G, hi = min(lo + G, nb);
    // 1. local suffixes of the group
    if (lo < hi) {
        double* cur = w.E[0];
        double* nxt = w.E[2];
        warp_copy<N>(agg + (size_t)(hi - 1) * ESZ, cur, lane);
        warp_store<N>(cur, suf + (size_t)(hi - 1) * ESZ, lane);
        for (int k = hi - 2; k >= lo; --k) {
            warp_copy<N>(agg + (size_t)k * ESZ, w.E[1], lane);
            warp_combine<N, M>(w.E[1], cur, nxt, w, lane);
            warp_store<N>(nxt, suf + (size_t)k * ESZ, lane);
            double* t = cur;
            cur = nxt;
            nxt = t;
        }
        warp_store<N>(cur, gbuf + (size_t)wl * ESZ, lane);
    }
    __syncthreads();
    // 2. suffix scan over the group aggregates
    double* gsrc = gbuf;
    double* gdst = gbuf + (size_t)RW_K2_WARPS * ESZ;
    for (int s = 1; s < ng; s <<= 1) {
        if (wl < ng) {
            if (wl + s < ng) {
                warp_copy<N>(gsrc + (size_t)wl * ESZ, w.E[0], lane);
                warp_copy<N>(gsrc + (size_t)(wl + s) * ESZ, w.E[1], lane);
                warp_combine<N, M>(w.E[0], w.E[1], w.E[2], w, lane);
                warp_store<N>(w.E[2], gdst + (size_t)wl * ESZ, lane);
            } else {
                for (int idx = lane; idx < ESZ; idx += 32)
                    gdst[(size_t)wl * ESZ + idx] = __ldcg(gsrc + (size_t)wl * ESZ + idx);
            }
        }
        __syncthreads();
        double* t = gsrc;
        gsrc = gdst;
        gdst = t;
    }
    // 3. complete the local suffixes with the next groups' suffix
    if (lo < hi && wl + 1 < ng) {
        warp_copy<N>(gsrc + (size_t)(wl + 1) * ESZ, w.E[1], lane);
        for (int k = lo; k < hi; ++k) {
            warp_copy<N>(suf + (size_t)k * ESZ, w.E[0], lane);
            warp_combine<N, M>(w.E[0], w.E[1], w.E[2], w, lane);
            warp_store<N>(w.E[2], suf + (size_t)k * ESZ, lane);
        }
    }
}

// K3: J after the chunk, then the information-form re-walk emitting the gains.
template <int N, int M, class Jac>
__device__ void riccati_k3(const Jac& jac, const RicArgs& p) {
    constexpr int ESZ = elemr_doubles<N>();
    constexpr int NN = N * N;
    extern __shared__ __align__(16) unsigned char rw_smem[];
    LqrShared<N, M>& sh = *reinterpret_cast<LqrShared<N, M>*>(rw_smem);
    RwWarp<N, M>* slices = reinterpret_cast<RwWarp<N, M>*>(rw_smem + sizeof(LqrShared<N, M>));
    lqr_shared_init<N, M>(sh, p.Q, p.R, p.dt);
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    RwWarp<N, M>& w = slices[wl];
    const int gw = blockIdx.x * RW_WARPS + wl;
    const int total = p.T + 1;
    const int lo = gw * p.L, hi = min(lo + p.L, total);
    if (lo >= total) return;
    const double* wsuf = p.agg + (size_t)(hs_rounds(RW_WARPS) & 1) * p.nwarp * ESZ;
    const double* bsuf = p.bagg + (size_t)p.nblk * ESZ;  // K2's output slot
    const bool next_warp = wl + 1 < RW_WARPS;
    const bool next_block = blockIdx.x + 1 < p.nblk;
    if (next_warp && next_block) {
        warp_copy<N>(wsuf + (size_t)(gw + 1) * ESZ, w.E[0], lane);
        warp_copy<N>(bsuf + (size_t)(blockIdx.x + 1) * ESZ, w.E[1], lane);
        warp_combine<N, M>(w.E[0], w.E[1], w.E[2], w, lane);
        for (int idx = lane; idx < NN; idx += 32) w.J2[idx] = w.E[2][2 * NN + idx];
    } else if (next_warp || next_block) {
        const double* sp = next_warp ? wsuf + (size_t)(gw + 1) * ESZ
                                     : bsuf + (size_t)(blockIdx.x + 1) * ESZ;
        for (int idx = lane; idx < NN; idx += 32) w.J2[idx] = __ldcg(sp + 2 * NN + idx);
    } else {
        for (int idx = lane; idx < NN; idx += 32) w.J2[idx] = 0.0;
    }
    __syncwarp();
    int local_fail = -1;
    const size_t TT = (size_t)p.T;
    for (int k = min(hi, p.T) - 1; k >= lo; --k) {
        warp_fg<N, M>(jac, k, p.dt, w, lane);
        // PG = P' G, PF = P' F with P' = J2 / 2 (PF kept in W's left half)
        for (int idx = lane; idx < N * M + NN; idx += 32) {
            if (idx < N * M) {
                const int i = idx / M, j = idx % M;
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < N; ++q) s += w.J2[i * N + q] * w.G[q * M + j];
                w.PG[idx] = 0.5 * s;
            } else {
                const int e2 = idx - N * M, i = e2 / N, j = e2 % N;
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < N; ++q) s += w.J2[i * N + q] * w.F[q * N + j];
                w.Tm[e2] = 0.5 * s;
            }
        }
        __syncwarp();
        // H = Rb + G' PG,  rhs = [G' PF | G']
        for (int idx = lane; idx < M * M + M * 2 * N; idx += 32) {
            if (idx < M * M) {
                const int i = idx / M, j = idx % M;
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < N; ++q) s += w.G[q * M + i] * w.PG[q * M + j];
                w.H[idx] = sh.Rb[i][j] + s;
            } else {
                const int e2 = idx - M * M, i = e2 / (2 * N), j = e2 % (2 * N);
                double s;
                if (j < N) {
                    s = 0.0;
#pragma unroll
                    for (int q = 0; q < N; ++q) s += w.G[q * M + i] * w.Tm[q * N + j];
                } else {
                    s = w.G[(j - N) * M + i];
                }
                w.rhs[e2] = s;
            }
        }
        __syncwarp();
        warp_gauss_jordan<M, 2 * N>(w.H, w.rhs, lane);  // rhs <- [K | H^-1 G']
        // outputs; Mt = I + C_k J2 with C_k = G Rt^-1 G'; W = F (Phi solve)
        for (int idx = lane; idx < M * N; idx += 32) {
            const int i = idx / N, j = idx % N;
            p.K[(size_t)idx * TT + k] = w.rhs[i * 2 * N + j];
            p.Lg[(size_t)idx * TT + k] = w.rhs[i * 2 * N + N + j];
        }
#if !FCB_RIC_GENERIC
        // Phi = (I + C_k J2)^-1 F equals Acl = F - G K (Woodbury with Rt = 2 Rb,
        // see warp_combine_base): no N x N solve
        for (int idx = lane; idx < NN; idx += 32) {
            const int i = idx / N;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < M; ++q) s += w.G[i * M + q] * w.rhs[q * 2 * N + idx % N];
            const double acl = w.F[idx] - s;
            p.Acl[(size_t)idx * TT + k] = acl;
            w.W[idx] = acl;
        }
        for (int idx = lane; idx < N * M; idx += 32) p.Gm[(size_t)idx * TT + k] = w.G[idx];
        __syncwarp();
#else
        for (int idx = lane; idx < NN; idx += 32) {
            const int i = idx / N, j = idx % N;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < M; ++q) s += w.G[i * M + q] * w.rhs[q * 2 * N + j];
            p.Acl[(size_t)idx * TT + k] = w.F[idx] - s;
            // C_k J2: C_k = G Rt^-1 G'
            double cj = (i == j) ? 1.0 : 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) {
                double c = 0.0;
#pragma unroll
                for (int a = 0; a < M; ++a) {
                    double gr = 0.0;
#pragma unroll
                    for (int r = 0; r < M; ++r) gr += w.G[i * M + r] * sh.Rtinv[r][a];
                    c += gr * w.G[q * M + a];
                }
                cj += c * w.J2[q * N + j];
            }
            w.Mt[idx] = cj;
            w.W[i * N + j] = w.F[idx];  // N x N right-hand side
        }
        for (int idx = lane; idx < N * M; idx += 32) p.Gm[(size_t)idx * TT + k] = w.G[idx];
        __syncwarp();
        warp_gauss_jordan<N, N>(w.Mt, w.W, lane);  // W <- Phi = (I + C J2)^-1 F
#endif
        // JF = J2 F (into JA), then J_k = Phi' JF + 2 Qb, symmetrised
        for (int idx = lane; idx < NN; idx += 32) {
            const int i = idx / N, j = idx % N;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += w.J2[i * N + q] * w.F[q * N + j];
            w.JA[idx] = s;
        }
        __syncwarp();
        for (int idx = lane; idx < NN; idx += 32) {
            const int i = idx / N, j = idx % N;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += w.W[q * N + i] * w.JA[q * N + j];
            w.Tm[idx] = s + 2.0 * sh.Qb[i][j];
        }
        __syncwarp();
        bool finite = true;
        for (int idx = lane; idx < NN; idx += 32) {
            const int i = idx / N, j = idx % N;
            const double v = 0.5 * (w.Tm[i * N + j] + w.Tm[j * N + i]);
            w.J2[idx] = v;
            finite = finite && isfinite(v);
        }
        finite = __all_sync(0xffffffffu, finite);
        __syncwarp();
        if (!finite && local_fail < 0) local_fail = k;
    }
    if (lane == 0 && local_fail >= 0) atomicMax(p.fail, local_fail);
}

// After kernel 3: publish a Riccati blow-up to the planner status word.
__device__ __forceinline__ void riccati_finish(const RicArgs& p) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int f = *((volatile int*)p.fail);
    if (f >= 0 && p.plan_state) {
        p.plan_state[FCB_STATE_STOP] = 2;
        p.plan_state[FCB_STATE_STAGE] = 3;
        p.plan_state[FCB_STATE_ITER] = p.iteration;
        p.plan_state[FCB_STATE_INDEX] = f;
    }
}

// Host: chunk length and grid of the Riccati phase for horizon T over
// `max_blocks` CTAs of RW_WARPS warps.
struct RicGeom {
    int L, nwarp, nblk;
};
inline RicGeom ric_geom(int T, int max_blocks) {
    const int total = T + 1;
    const long cap = (long)max_blocks * RW_WARPS;
    int L = (int)std::max<long>(RW_MIN_CHUNK, (total + cap - 1) / cap);
    const int used = (total + L - 1) / L;
    const int nblk = (used + RW_WARPS - 1) / RW_WARPS;
    return RicGeom{L, nblk * RW_WARPS, nblk};
}

}  // namespace fcb
