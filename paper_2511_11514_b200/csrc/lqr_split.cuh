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

// Riccati-phase launch geometry: RIC_BLOCK threads per CTA, each thread owns
// a chunk of `L` consecutive elements (the zero terminal element T included).
constexpr int RIC_BLOCK = 128;
constexpr int RIC_MIN_CHUNK = 4;

struct RicArgs {
    int T;
    double dt;
    const double* Q;
    const double* R;
    int L;        // elements per thread chunk
    int nthr;     // threads with a chunk slot (nblk * RIC_BLOCK)
    int nblk;     // CTAs of the thread-level kernels
    double* agg;  // 2 * nthr * 3N^2: chunk aggregates -> in-CTA suffixes (ping-pong)
    double* bagg; // 2 * nblk * 3N^2: CTA aggregates -> their suffix scan (ping-pong)
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

template <int N>
__device__ __forceinline__ void elemr_identity(ElemR<N>& e) {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            e.A[i][j] = (i == j) ? 1.0 : 0.0;
            e.C[i][j] = 0.0;
            e.J[i][j] = 0.0;
        }
}

// F = I + dt A_k, G = dt B_k at step k and the base element
// e_k = (F, G Rt^-1 G', 2 Qb); the terminal element (k >= T) is zero.
template <int N, int M, class Jac>
struct RicSteps {
    const Jac& jac;
    const LqrShared<N, M>& sh;
    int T;
    double dt;
    __device__ __forceinline__ void fg(int k, double (&F)[N][N], double (&G)[N][M]) const {
        double a[N * N], b[N * M];
        jac.get(k, a, b);
#pragma unroll
        for (int i = 0; i < N; ++i) {
#pragma unroll
            for (int j = 0; j < N; ++j) F[i][j] = (i == j ? 1.0 : 0.0) + dt * a[i * N + j];
#pragma unroll
            for (int j = 0; j < M; ++j) G[i][j] = dt * b[i * M + j];
        }
    }
    __device__ __forceinline__ void base(int k, ElemR<N>& e) const {
        if (k >= T) {
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
                for (int j = 0; j < N; ++j) e.A[i][j] = e.C[i][j] = e.J[i][j] = 0.0;
            return;
        }
        double F[N][N], G[N][M];
        fg(k, F, G);
        base_fg(F, G, e);
    }
    __device__ __forceinline__ void base_fg(const double (&F)[N][N], const double (&G)[N][M],
                                            ElemR<N>& e) const {
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
    }
};

// Riccati phase, kernel 1 of 3: every thread folds its chunk of elements into
// one aggregate (suffix order), then the CTA runs an inclusive Hillis-Steele
// suffix scan over its threads' aggregates.  Threads past the last element
// hold the identity.
template <int N, int M, class Jac>
__device__ void riccati_k1(const Jac& jac, const RicArgs& p) {
    constexpr int ESZ = elemr_doubles<N>();
    __shared__ LqrShared<N, M> sh;
    lqr_shared_init<N, M>(sh, p.Q, p.R, p.dt);
    const RicSteps<N, M, Jac> st{jac, sh, p.T, p.dt};
    const int t = blockIdx.x * RIC_BLOCK + threadIdx.x;
    const int total = p.T + 1;
    const int lo = t * p.L, hi = min(lo + p.L, total);
    if (t == 0) *p.fail = -1;
    ElemR<N> acc;
    if (lo < total) {
        ElemR<N> e, tmp;
        st.base(hi - 1, acc);
        for (int k = hi - 2; k >= lo; --k) {
            st.base(k, e);
            elemr_combine<N>(e, acc, tmp);
            acc = tmp;
        }
    } else {
        elemr_identity<N>(acc);
    }
    double* src = p.agg;
    double* dst = p.agg + (size_t)p.nthr * ESZ;
    elemr_store<N>(src + (size_t)t * ESZ, acc);
    __syncthreads();
    for (int s = 1; s < RIC_BLOCK; s <<= 1) {
        if (threadIdx.x + s < RIC_BLOCK) {
            ElemR<N> b, o;
            elemr_load<N>(src + (size_t)(t + s) * ESZ, b);
            elemr_combine<N>(acc, b, o);
            acc = o;
        }
        elemr_store<N>(dst + (size_t)t * ESZ, acc);
        __syncthreads();
        double* tt = src;
        src = dst;
        dst = tt;
    }
    // the CTA aggregate (suffix of its first thread) feeds kernel 2
    if (threadIdx.x == 0) elemr_store<N>(p.bagg + (size_t)blockIdx.x * ESZ, acc);
}

// Kernel 2 of 3 (one CTA): inclusive suffix scan over the CTA aggregates.
template <int N>
__device__ void riccati_k2(const RicArgs& p) {
    constexpr int ESZ = elemr_doubles<N>();
    double* src = p.bagg;
    double* dst = p.bagg + (size_t)p.nblk * ESZ;
    const int b = threadIdx.x;
    for (int s = 1; s < p.nblk; s <<= 1) {
        if (b < p.nblk) {
            ElemR<N> a;
            elemr_load<N>(src + (size_t)b * ESZ, a);
            if (b + s < p.nblk) {
                ElemR<N> c, o;
                elemr_load<N>(src + (size_t)(b + s) * ESZ, c);
                elemr_combine<N>(a, c, o);
                elemr_store<N>(dst + (size_t)b * ESZ, o);
            } else {
                elemr_store<N>(dst + (size_t)b * ESZ, a);
            }
        }
        __syncthreads();
        double* tt = src;
        src = dst;
        dst = tt;
    }
}

// Kernel 3 of 3: each thread forms J_{hi} (the value matrix after its chunk)
// from the in-CTA suffix of the next thread and the suffix of the next CTAs,
// then re-walks its chunk in information form emitting the gains.
template <int N, int M, class Jac>
__device__ void riccati_k3(const Jac& jac, const RicArgs& p) {
    constexpr int ESZ = elemr_doubles<N>();
    __shared__ LqrShared<N, M> sh;
    lqr_shared_init<N, M>(sh, p.Q, p.R, p.dt);
    const RicSteps<N, M, Jac> st{jac, sh, p.T, p.dt};
    const int t = blockIdx.x * RIC_BLOCK + threadIdx.x;
    const int total = p.T + 1;
    const int lo = t * p.L, hi = min(lo + p.L, total);
    if (lo >= total) return;
    const double* tsuf = p.agg + (size_t)(hs_rounds(RIC_BLOCK) & 1) * p.nthr * ESZ;
    const double* bsuf = p.bagg + (size_t)(hs_rounds(p.nblk) & 1) * p.nblk * ESZ;
    const bool next_thread = threadIdx.x + 1 < RIC_BLOCK;
    const bool next_block = blockIdx.x + 1 < p.nblk;
    double J2[N][N];
    if (next_thread && next_block) {
        ElemR<N> a, b, o;
        elemr_load<N>(tsuf + (size_t)(t + 1) * ESZ, a);
        elemr_load<N>(bsuf + (size_t)(blockIdx.x + 1) * ESZ, b);
        elemr_combine<N>(a, b, o);
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
            for (int j = 0; j < N; ++j) J2[i][j] = o.J[i][j];
    } else if (next_thread || next_block) {
        const double* sp = next_thread ? tsuf + (size_t)(t + 1) * ESZ
                                       : bsuf + (size_t)(blockIdx.x + 1) * ESZ;
#pragma unroll
        for (int i = 0; i < N * N; ++i) (&J2[0][0])[i] = __ldcg(sp + 2 * N * N + i);
    } else {
#pragma unroll
        for (int i = 0; i < N * N; ++i) (&J2[0][0])[i] = 0.0;
    }
    int local_fail = -1;
    for (int k = hi - 1; k >= lo; --k) {
        if (k >= p.T) continue;
        double F[N][N], G[N][M];
        st.fg(k, F, G);
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
                    const double tq = H[col][q];
                    H[col][q] = H[pv][q];
                    H[pv][q] = tq;
                }
#pragma unroll
                for (int q = 0; q < 2 * N; ++q) {
                    const double tq = rhs[col][q];
                    rhs[col][q] = rhs[pv][q];
                    rhs[pv][q] = tq;
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
        st.base_fg(F, G, e);
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
    if (local_fail >= 0) atomicMax(p.fail, local_fail);
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
// `max_blocks` CTAs.
struct RicGeom {
    int L, nthr, nblk;
};
inline RicGeom ric_geom(int T, int max_blocks) {
    const int total = T + 1;
    const long cap = (long)max_blocks * RIC_BLOCK;
    int L = (int)std::max<long>(RIC_MIN_CHUNK, (total + cap - 1) / cap);
    const int used = (total + L - 1) / L;
    const int nblk = (used + RIC_BLOCK - 1) / RIC_BLOCK;
    return RicGeom{L, nblk * RIC_BLOCK, nblk};
}

}  // namespace fcb
