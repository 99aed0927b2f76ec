// stein_dev.cuh -- device pieces of the Stein flow shared by the per-iteration
// kernels (stein.cu) and the persistent Stein planner (plan_stein.cuh).
#pragma once

#include "fcb_internal.cuh"

namespace fcb {

constexpr double BANDWIDTH_FLOOR = 1e-12;  // stein.py:34

// GaussianMixture score and log density at one point (reference.py:77-110):
// per component the Cholesky solves of Sigma^-1 (x - mu), responsibilities by
// a running log-sum-exp.  prm = [log_w(k) | log_norm(k) | mu(k D) | chol(k D D)].
template <int D>
__device__ __forceinline__ void gmm_point(const double* __restrict__ xp, int k,
                                          const double* __restrict__ prm, double* score,
                                          double* logdens) {
    const double* logw = prm;
    const double* lognorm = prm + k;
    const double* mu = prm + 2 * k;
    const double* chol = prm + 2 * k + (size_t)k * D;
    double x[D];
#pragma unroll
    for (int q = 0; q < D; ++q) x[q] = xp[q];
    double M = -INFINITY, S = 0.0, acc[D];
#pragma unroll
    for (int q = 0; q < D; ++q) acc[q] = 0.0;
    for (int c = 0; c < k; ++c) {
        const double* L = chol + (size_t)c * D * D;
        double diff[D], y[D], pull[D];
#pragma unroll
        for (int q = 0; q < D; ++q) diff[q] = x[q] - mu[(size_t)c * D + q];
        // forward substitution L y = diff
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double v = diff[r];
#pragma unroll
            for (int q = 0; q < r; ++q) v -= L[r * D + q] * y[q];
            y[r] = v / L[r * D + r];
        }
        // back substitution L^T pull = y
#pragma unroll
        for (int r = D - 1; r >= 0; --r) {
            double v = y[r];
#pragma unroll
            for (int q = r + 1; q < D; ++q) v -= L[q * D + r] * pull[q];
            pull[r] = v / L[r * D + r];
        }
        double quad = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) quad += diff[q] * pull[q];
        const double sc = -0.5 * quad - lognorm[c] + logw[c];
        if (sc > M) {
            const double r = (S > 0.0) ? exp(M - sc) : 0.0;
            S = S * r + 1.0;
#pragma unroll
            for (int q = 0; q < D; ++q) acc[q] = acc[q] * r + pull[q];
            M = sc;
        } else {
            const double r = exp(sc - M);
            S += r;
#pragma unroll
            for (int q = 0; q < D; ++q) acc[q] += r * pull[q];
        }
    }
    if (score) {
#pragma unroll
        for (int q = 0; q < D; ++q) score[q] = -acc[q] / S;
    }
    if (logdens) *logdens = M + log(S);
}

template <int D>
__device__ __forceinline__ unsigned long long sqdist_key(const double* a, const double* b) {
    // (a0-b0)^2 + (a1-b1)^2 [+ (a2-b2)^2], left to right, no contraction
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
        const double df = __dsub_rn(a[q], b[q]);
        const double sq = __dmul_rn(df, df);
        acc = (q == 0) ? sq : __dadd_rn(acc, sq);
    }
    return (unsigned long long)__double_as_longlong(acc);
}

// radix passes of the exact median: 11-bit digits from the top, the last 8 bits
__device__ __forceinline__ int med_pass_shift(int pass) { return pass < 5 ? 52 - 11 * pass : 0; }
__device__ __forceinline__ int med_pass_bits(int pass) { return pass < 5 ? 11 : 8; }

// h = med^2 / log(n+1) from the two selected order statistics (stein.py:66-76):
// np.median averages the middle pair when n^2 is even.
__device__ __forceinline__ void median_finish_vals(unsigned long long klo_bits,
                                                   unsigned long long khi_bits, int n,
                                                   double log_np1, double* hstat) {
    const double vlo = __longlong_as_double((long long)klo_bits);
    const double vhi = __longlong_as_double((long long)khi_bits);
    const unsigned long long N = (unsigned long long)n * (unsigned long long)n;
    double med;
    if (N % 2ull == 1ull) med = sqrt(vlo);
    else med = __ddiv_rn(__dadd_rn(sqrt(vlo), sqrt(vhi)), 2.0);
    double h = __ddiv_rn(__dmul_rn(med, med), log_np1);
    const bool clamped = h <= BANDWIDTH_FLOOR;
    if (clamped) h = BANDWIDTH_FLOOR;
    hstat[0] = h;
    hstat[1] = med;
    hstat[2] = clamped ? 1.0 : 0.0;
    hstat[3] = 0.0;
}

}  // namespace fcb
