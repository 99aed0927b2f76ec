// plan_scan.cuh -- the planner's per-iteration time recurrences as affine scans
// (affscan.cuh): the linear-model rollout and the two passes of the LQR
// affine phase (lqr_split.cuh), each with its outputs fused into the scan's
// consumer.
#pragma once

#include "affscan.cuh"
#include "fcb_internal.cuh"

namespace fcb {

// ---------------------------------------------------------------------------
// LQR affine phase
// ---------------------------------------------------------------------------
// The Riccati outputs are element-major (X[e * T + k], lqr_split.cuh), so a
// warp reading one element of 32 consecutive steps is one coalesced load.
//
// backward: eta_k = Acl_k' eta_{k+1} + 2 Qb a_k  (eta = -2 p of lqr.py:190,
// with the reference's closed = F - G K)
template <int N, class Flow>
struct EtaMap {
    const double* Acl;
    const double* Q;
    double dt;
    int T;
    Flow flow;
    __device__ void operator()(int k, AMap<N>& m) const {
        double ak[N];
        flow.get(k, ak);
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) s += Q[i * N + q] * ak[q];
            m.c[i] = 2.0 * dt * s;
#pragma unroll
            for (int j = 0; j < N; ++j) m.M[i][j] = Acl[(size_t)(j * N + i) * T + k];
        }
    }
};

// consumer: d_k = 1/2 Lg_k eta_{k+1}; the first non-finite eta index
template <int N, int M>
struct EtaOut {
    const double* Lg;
    double* dff;
    int* fail;
    int T;
    __device__ double operator()(int k, const double* e_next, const double* e_k) const {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) s += Lg[(size_t)(i * N + j) * T + k] * e_next[j];
            dff[(size_t)k * M + i] = 0.5 * s;
        }
        bool finite = true;
#pragma unroll
        for (int i = 0; i < N; ++i) finite = finite && isfinite(e_k[i]);
        if (!finite) atomicMax(fail, k);
        return 0.0;
    }
};

// forward: z_{k+1} = Acl_k z_k + G_k d_k
template <int N, int M>
struct ZMap {
    const double* Acl;
    const double* Gm;
    const double* dff;
    int T;
    __device__ void operator()(int k, AMap<N>& m) const {
        double dk[M];
#pragma unroll
        for (int i = 0; i < M; ++i) dk[i] = dff[(size_t)k * M + i];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double cc = 0.0;
#pragma unroll
            for (int q = 0; q < M; ++q) cc += Gm[(size_t)(i * M + q) * T + k] * dk[q];
            m.c[i] = cc;
#pragma unroll
            for (int j = 0; j < N; ++j) m.M[i][j] = Acl[(size_t)(i * N + j) * T + k];
        }
    }
};

// consumer: v_k = d_k - K_k z_k, the stage cost, z, the control update
template <int N, int M, class Flow>
struct ZOut {
    const double* K;  // element-major
    int T;
    const double* dff;
    const double* Q;
    const double* R;
    double dt;
    Flow flow;
    const int* fail;
    double* v;
    double* z;
    const double* U;
    double* U_next;
    double eta;
    const double* clamp;
    __device__ double operator()(int k, const double* zk, const double* zk1) const {
        if (*((volatile const int*)fail) >= 0) return 0.0;
        double vk[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) s += K[(size_t)(i * N + j) * T + k] * zk[j];
            vk[i] = dff[(size_t)k * M + i] - s;
        }
        double ak[N], e[N];
        flow.get(k, ak);
#pragma unroll
        for (int i = 0; i < N; ++i) e[i] = ak[i] - zk[i];
        double c1 = 0.0, c2 = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) s += (dt * Q[i * N + j]) * e[j];
            c1 += e[i] * s;
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < M; ++j) s += (dt * R[i * M + j]) * vk[j];
            c2 += vk[i] * s;
        }
        if (v)
#pragma unroll
            for (int i = 0; i < M; ++i) v[(size_t)k * M + i] = vk[i];
        if (z) {
            if (k == 0)
#pragma unroll
                for (int i = 0; i < N; ++i) z[i] = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) z[(size_t)(k + 1) * N + i] = zk1[i];
        }
        if (U_next)
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double u = U[(size_t)k * M + i] + eta * vk[i];
                if (clamp) u = fmin(fmax(u, -clamp[i]), clamp[i]);
                U_next[(size_t)k * M + i] = u;
            }
        return c1 + c2;
    }
};

// After both scans: total cost, status, planner hooks.
__device__ __forceinline__ void lqr_finish_body(double total, int* fail, double* cost,
                                                double* lqr_costs, int* plan_state, int iteration) {
    const int f = *((volatile int*)fail);
    if (f >= 0) {
        if (plan_state) {
            plan_state[FCB_STATE_STOP] = 2;
            plan_state[FCB_STATE_STAGE] = 3;
            plan_state[FCB_STATE_ITER] = iteration;
            plan_state[FCB_STATE_INDEX] = f;
        }
        return;
    }
    if (cost) *cost = total;
    if (plan_state) {
        lqr_costs[iteration] = total;
        plan_state[FCB_STATE_UPDATES] = iteration + 1;
    }
}

__global__ void lqr_finish_kernel(int nb, const double* red, int* fail, double* cost,
                                  double* lqr_costs, int* plan_state, int iteration, int gated) {
    if (threadIdx.x != 0) return;
    if (gated && plan_state && *((volatile int*)plan_state) != 0) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += red[b];
    lqr_finish_body(s, fail, cost, lqr_costs, plan_state, iteration);
}

// Flag slots of the one-launch kernels (per launch tag, AS_BLK flags each).
struct FusedWs {
    double* agg0;      // FUSED_MAX_BLOCKS maps (N <= 6)
    double* agg1;
    double* vals;      // FUSED_MAX_BLOCKS
    int* ivals;        // FUSED_MAX_BLOCKS
    unsigned* flags;   // 4 * AS_BLK
};

// The whole affine phase in one launch for T <= AS_BLK^2: eta scan (emits d),
// the blocks' eta status, z scan (v, cost, z, U update) and the finish.
template <int N, int M, class Flow>
__global__ void __launch_bounds__(AS_BLK)
    affine_fused_kernel(int T, EtaMap<N, Flow> emap, EtaOut<N, M> eout, ZMap<N, M> zmap,
                        ZOut<N, M, Flow> zout, FusedWs fw, unsigned tag, int* fail, int reset_fail,
                        double* cost, double* lqr_costs, int* plan_state, int iteration) {
    extern __shared__ double sbuf[];
    __shared__ ScanShared<N> sh;
    __shared__ int s_fail_eta, s_fail_all;
    __shared__ double s_tmp[AS_BLK];
    if (plan_state && *((volatile int*)plan_state) != 0) return;
    FCB_SCAN_MARK(0);
    const int t = threadIdx.x;
    if (t == 0) {
        s_fail_eta = -1;
        s_fail_all = reset_fail ? -1 : *((volatile int*)fail);
    }
    __syncthreads();
    EtaOut<N, M> eo = eout;
    eo.fail = &s_fail_eta;
    fused_scan<N, false>(T, emap, eo, nullptr, fw.agg0, fw.flags, tag, sbuf, sh);
    if (t == 0) {
        fw.ivals[blockIdx.x] = s_fail_eta;
        __threadfence();
        st_release_flag(fw.flags + AS_BLK + blockIdx.x, tag);
    }
    // the z consumer skips every step once any eta is non-finite: every
    // block's eta status is gathered during the z look-back
    ZOut<N, M, Flow> zo = zout;
    zo.fail = &s_fail_all;
    const ExtraWait xw{fw.flags + AS_BLK, fw.ivals, &s_fail_all, tag};
    const double part = fused_scan<N, true>(T, zmap, zo, nullptr, fw.agg1, fw.flags + 2 * AS_BLK,
                                            tag, sbuf, sh, &xw);
    publish_value(fw.vals, fw.flags + 3 * AS_BLK, tag, part);
    if (blockIdx.x == 0) {
        const double total = gather_sum(fw.vals, fw.flags + 3 * AS_BLK, tag, s_tmp);
        if (t == 0) {
            *fail = s_fail_all;
            lqr_finish_body(total, fail, cost, lqr_costs, plan_state, iteration);
        }
    }
    FCB_SCAN_MARK(9);
}

// ---------------------------------------------------------------------------
// linear-model rollout:  s_{k+1} = Phi s_k + Gam u_k
// ---------------------------------------------------------------------------
template <int N, int M>
struct RollMap {
    const double* PhiGam;  // [Phi (N*N) | Gam (N*M)]
    const double* U;
    __device__ void operator()(int k, AMap<N>& m) const {
        double u[M];
#pragma unroll
        for (int j = 0; j < M; ++j) u[j] = U[(size_t)k * M + j];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < M; ++j) s += PhiGam[N * N + i * M + j] * u[j];
            m.c[i] = s;
#pragma unroll
            for (int j = 0; j < N; ++j) m.M[i][j] = PhiGam[i * N + j];
        }
    }
};

template <class Mdl>
struct RollOut {
    static constexpr int N = Mdl::N;
    double* S;
    const double* s0;
    double* X;
    const double* P;
    int d;
    int* first_bad;
    const double* prm;
    const double* U;
    double dt;
    __device__ double operator()(int k, const double* sk, const double* sk1) const {
        if (k == 0)
#pragma unroll
            for (int i = 0; i < N; ++i) S[i] = s0[i];
        bool finite = true;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            S[(size_t)(k + 1) * N + i] = sk1[i];
            finite = finite && isfinite(sk1[i]);
        }
        {
            // the reference's step from s_k, stage by stage: an overflow in an
            // intermediate stage marks the same step the sequential RK4 does
            double u[Mdl::M], k1[N], k2[N], k3[N], k4[N], t[N];
#pragma unroll
            for (int j = 0; j < Mdl::M; ++j) u[j] = U[(size_t)k * Mdl::M + j];
            const double half = __dmul_rn(0.5, dt), sixth = dt / 6.0;
            Mdl::f(sk, u, prm, k1);
#pragma unroll
            for (int j = 0; j < N; ++j) t[j] = __dadd_rn(sk[j], __dmul_rn(half, k1[j]));
            Mdl::f(t, u, prm, k2);
#pragma unroll
            for (int j = 0; j < N; ++j) t[j] = __dadd_rn(sk[j], __dmul_rn(half, k2[j]));
            Mdl::f(t, u, prm, k3);
#pragma unroll
            for (int j = 0; j < N; ++j) t[j] = __dadd_rn(sk[j], __dmul_rn(dt, k3[j]));
            Mdl::f(t, u, prm, k4);
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double inner = __dadd_rn(__dadd_rn(k1[j], __dmul_rn(2.0, __dadd_rn(k2[j], k3[j]))), k4[j]);
                finite = finite && isfinite(__dadd_rn(sk[j], __dmul_rn(sixth, inner)));
            }
        }
        if (X)
            for (int r = 0; r < d; ++r) {
                double a = 0.0;
#pragma unroll
                for (int j = 0; j < N; ++j) a += sk1[j] * P[r * N + j];
                X[(size_t)k * d + r] = a;
            }
        if (!finite) atomicMin(first_bad, k + 1);
        return 0.0;
    }
};

// ---------------------------------------------------------------------------
// triangular models (diff_drive, aircraft_3d): the integrator states q obey
// q' = qdot(u) and the positions p' = pdot(q, u), so one RK4/ZOH step is
//   q_{k+1} = q_k + dt/6 (qd + 2 (qd + qd) + qd)
//   p_{k+1} = p_k + dt/6 (k1 + 2 (k2 + k3) + k4),  k_i = pdot(q at stage i)
// with stage values of q known in closed form.  Exact RK4 stage arithmetic
// (the reference's operation order per step); only the accumulation over
// steps is a prefix sum.
// ---------------------------------------------------------------------------
template <class Mdl>
__device__ __forceinline__ void tri_qinc(const double* u, double dt, double* dq) {
    double qd[Mdl::NQ];
    Mdl::qdot(u, qd);
    const double sixth = dt / 6.0;
#pragma unroll
    for (int i = 0; i < Mdl::NQ; ++i) {
        const double inner = __dadd_rn(__dadd_rn(qd[i], __dmul_rn(2.0, __dadd_rn(qd[i], qd[i]))), qd[i]);
        dq[i] = __dmul_rn(sixth, inner);
    }
}

template <class Mdl>
__device__ __forceinline__ void tri_pinc(const double* q, const double* u, double dt, double* dp) {
    constexpr int NQ = Mdl::NQ, NP = Mdl::NP;
    double qd[NQ], qs[NQ], k1[NP], k2[NP], k3[NP], k4[NP];
    Mdl::qdot(u, qd);
    const double half = __dmul_rn(0.5, dt), sixth = dt / 6.0;
    Mdl::pdot(q, u, k1);
#pragma unroll
    for (int i = 0; i < NQ; ++i) qs[i] = __dadd_rn(q[i], __dmul_rn(half, qd[i]));
    Mdl::pdot(qs, u, k2);
    Mdl::pdot(qs, u, k3);  // k3's q stage equals k2's (qd is constant over the step)
#pragma unroll
    for (int i = 0; i < NQ; ++i) qs[i] = __dadd_rn(q[i], __dmul_rn(dt, qd[i]));
    Mdl::pdot(qs, u, k4);
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        const double inner = __dadd_rn(__dadd_rn(k1[i], __dmul_rn(2.0, __dadd_rn(k2[i], k3[i]))), k4[i]);
        dp[i] = __dmul_rn(sixth, inner);
    }
}

template <class Mdl>
struct TriQMap {
    const double* U;
    double dt;
    __device__ void operator()(int k, AMap<Mdl::NQ>& m) const {
        double u[Mdl::M];
#pragma unroll
        for (int j = 0; j < Mdl::M; ++j) u[j] = U[(size_t)k * Mdl::M + j];
        tri_qinc<Mdl>(u, dt, m.c);
#pragma unroll
        for (int i = 0; i < Mdl::NQ; ++i)
#pragma unroll
            for (int j = 0; j < Mdl::NQ; ++j) m.M[i][j] = (i == j) ? 1.0 : 0.0;
    }
};

// consumer of the q scan: q into S, the position increment into dp
template <class Mdl>
struct TriQOut {
    const double* U;
    double dt;
    double* S;
    const double* s0;
    double* dp;  // T x NP
    int* first_bad;
    __device__ double operator()(int k, const double* qk, const double* qk1) const {
        constexpr int N = Mdl::N;
        if (k == 0)
            for (int i = 0; i < N; ++i) S[i] = s0[i];
        double u[Mdl::M];
#pragma unroll
        for (int j = 0; j < Mdl::M; ++j) u[j] = U[(size_t)k * Mdl::M + j];
        tri_pinc<Mdl>(qk, u, dt, dp + (size_t)k * Mdl::NP);
        bool finite = true;
#pragma unroll
        for (int i = 0; i < Mdl::NQ; ++i) {
            S[(size_t)(k + 1) * N + Mdl::QOFF + i] = qk1[i];
            finite = finite && isfinite(qk1[i]);
        }
        if (!finite) atomicMin(first_bad, k + 1);
        return 0.0;
    }
};

template <class Mdl>
struct TriPMap {
    const double* dp;
    __device__ void operator()(int k, AMap<Mdl::NP>& m) const {
#pragma unroll
        for (int i = 0; i < Mdl::NP; ++i) {
            m.c[i] = dp[(size_t)k * Mdl::NP + i];
#pragma unroll
            for (int j = 0; j < Mdl::NP; ++j) m.M[i][j] = (i == j) ? 1.0 : 0.0;
        }
    }
};

// consumer of the p scan: positions into S, the workspace projection into X
template <class Mdl>
struct TriPOut {
    double* S;
    double* X;
    const double* P;
    int d;
    int* first_bad;
    __device__ double operator()(int k, const double*, const double* pk1) const {
        constexpr int N = Mdl::N;
        bool finite = true;
#pragma unroll
        for (int i = 0; i < Mdl::NP; ++i) {
            S[(size_t)(k + 1) * N + i] = pk1[i];
            finite = finite && isfinite(pk1[i]);
        }
        if (X) {
            // X = P s_{k+1}; read the q part written by the q scan
            for (int r = 0; r < d; ++r) {
                double a = 0.0;
                for (int j = 0; j < N; ++j) {
                    const double sj = (j < Mdl::NP) ? pk1[j] : S[(size_t)(k + 1) * N + j];
                    a += sj * P[r * N + j];
                }
                X[(size_t)k * d + r] = a;
            }
        }
        if (!finite) atomicMin(first_bad, k + 1);
        return 0.0;
    }
};

// first_bad starts at 0x7f7f7f7f (byte memset): no non-finite state seen
__device__ __forceinline__ void roll_finish_body(int first_bad, int* status, int* plan_state,
                                                 int iteration) {
    const int f = (first_bad >= 0x7f7f7f7f) ? -1 : first_bad;
    if (status) *status = f;
    if (plan_state && f >= 0) {
        plan_state[FCB_STATE_STOP] = 2;
        plan_state[FCB_STATE_STAGE] = 1;
        plan_state[FCB_STATE_ITER] = iteration;
        plan_state[FCB_STATE_INDEX] = f;
    }
}

__global__ void roll_finish_kernel(int* first_bad, int* status, int* plan_state, int iteration) {
    if (threadIdx.x != 0) return;
    if (plan_state && *((volatile int*)plan_state) != 0) return;
    roll_finish_body(*first_bad, status, plan_state, iteration);
}

}  // namespace fcb
