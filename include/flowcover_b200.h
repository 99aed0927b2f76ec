/*
 * flowcover_b200.h -- C ABI of the B200-native reference-flow generator.
 *
 * Drop-in boundary for the hot path of the reference package `flowcover`
 * (/root/reference/pkg/src/flowcover).  Each entry point below replaces one
 * reference Python function; the citation names the function it replaces.
 * The Python layer (paper_2511_11514_b200/*.py) keeps the reference's public
 * signatures and binds these symbols with ctypes.
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer owned by the caller unless
 *     documented otherwise; calls are stream-ordered on `stream` (a
 *     cudaStream_t passed as void*) and never synchronize the device.
 *   - Point sets are row-major float64 (rows, d) with d in {1, 2, 3}.
 *   - Scratch memory is caller-provided (`ws`, `ws_bytes`); size it with the
 *     matching *_workspace_bytes query.  Calls do not allocate.
 *   - Scalars produced on device (omega, err, iteration counts, bandwidths)
 *     are written to device memory so a planning loop never round-trips.
 *   - `gate` (nullable): a device int; when *gate != 0 at kernel start the
 *     call is a no-op.  The planner uses it to stop a queued loop on device.
 *   - Return value: FCB_OK or an FCB_E* status; fcb_last_error() explains.
 *     Algorithmic failures discovered on device (rollout blow-up, Riccati
 *     blow-up, transport marginal violation) are reported through device
 *     status words, mirroring the reference's typed exceptions.
 */
#ifndef FLOWCOVER_B200_H
#define FLOWCOVER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* fcb_stream_t; /* cudaStream_t */

#if defined(__GNUC__)
#define FCB_API __attribute__((visibility("default")))
#else
#define FCB_API
#endif

enum {
    FCB_OK = 0,
    FCB_EINPUT = 1,     /* ValueError / SinkhornInputError              */
    FCB_EFLOW = 2,      /* FlowError          (sinkhorn.py:74-75)        */
    FCB_EROLLOUT = 3,   /* RolloutDivergenceError (dynamics.py:25-30)    */
    FCB_ERICCATI = 4,   /* RiccatiDivergenceError (lqr.py:47-55)         */
    FCB_ECUDA = 5,
    FCB_ENOTSUP = 6,
    FCB_EWORKSPACE = 7
};

enum { FCB_FP32 = 0, FCB_FP64 = 1 };

/* Dynamics models with device implementations (dynamics.py:72-181). */
enum {
    FCB_MODEL_SINGLE_INTEGRATOR_2D = 0, /* dynamics.py:72-95            */
    FCB_MODEL_DIFF_DRIVE = 1,           /* dynamics.py:98-129           */
    FCB_MODEL_AIRCRAFT_3D = 2,          /* dynamics.py:132-181          */
    FCB_MODEL_DOUBLE_INTEGRATOR_2D = 3, /* user-built model of SURVEY §8(d) cfg 1-2 */
    FCB_MODEL_LTI = 4                   /* f = A s + B u, A/B in model_params */
};

/* Entropic-OT solve modes (sinkhorn.py:170-236). */
enum { FCB_OT_ASYM = 0, FCB_OT_SYM = 1, FCB_OT_SWEEP = 2 };

/* Planner status words (device int[8]); see fcb_plan_state_* below. */
enum {
    FCB_STATE_STOP = 0,      /* 0 running, 1 converged, 2 failed          */
    FCB_STATE_STAGE = 1,     /* 1 rollout, 2 flow, 3 lqr                  */
    FCB_STATE_ITER = 2,      /* outer iteration of the failure            */
    FCB_STATE_INDEX = 3,     /* rollout step / Riccati index              */
    FCB_STATE_FLOWS = 4,     /* flows evaluated (iterations_used)         */
    FCB_STATE_UPDATES = 5    /* control updates applied                   */
};

/* ---- library ----------------------------------------------------------- */
FCB_API const char* fcb_version(void);
FCB_API const char* fcb_last_error(void);
FCB_API long long fcb_launch_count(void); /* kernels launched by this library      */
FCB_API const char* fcb_last_kernel(void); /* name of the last kernel launched (tests) */
FCB_API int fcb_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---- entropic OT / Sinkhorn (sinkhorn.py) ------------------------------ */

/* resolve_omega (sinkhorn.py:136-148) plus the centring statistics the
 * kernels use.  omega_fixed > 0 selects a numeric omega, otherwise "auto".
 * scal: device double[16]; scal[0] = omega.  mode picks the centre
 * (ASYM: midpoint of the means, SYM: mean of X). */
FCB_API size_t fcb_omega_workspace_bytes(int n, int m);
FCB_API int fcb_resolve_omega(int mode, const double* X, int n, const double* Y, int m, int d,
                      double omega_fixed, double* scal, void* ws, size_t ws_bytes,
                      fcb_stream_t stream);

/* One transport solve with streamed cost tiles; the n x m cost matrix is
 * never stored.
 *   ASYM  : _solve_asymmetric (sinkhorn.py:170-205) on X (n) vs Y (m)
 *   SYM   : _solve_symmetric  (sinkhorn.py:208-236) on X (n); Y ignored
 *   SWEEP : one _lse_rows sweep (sinkhorn.py:151-167):
 *           f[i] = LSE_j((f0[j] - |x_i - y_j|^2) / omega), f0 has m entries
 * scal     : from fcb_resolve_omega.
 * f0       : nullable warm start (n), or the SWEEP potential (m).
 * f, g     : potentials out (g: m, ASYM only; may be NULL otherwise).
 * row_sums : plan row sums exp(clip(delta) + log a) (n).
 * stat     : device double[4] = {marginal_error, iters_used, converged, 0}.
 * bary     : nullable (n*(d+1)): per row the unclipped plan row mass and
 *            plan barycentre, i.e. sum_j T_ij and sum_j T_ij y_j / sum_j T_ij
 *            at the returned potentials (feeds the transport gradient,
 *            sinkhorn.py:383-391).  In SWEEP mode: {1, weighted mean of
 *            the columns under the sweep's softmax weights} per row, which
 *            is what an M-sharded caller needs to combine shards. */
FCB_API size_t fcb_ot_workspace_bytes(int mode, int precision, int n, int m, int d);
FCB_API int fcb_ot_solve(int mode, int precision, const double* X, int n, const double* Y, int m, int d,
                 const double* scal, int max_iters, double tol, const double* f0,
                 double* f, double* g, double* row_sums, double* stat, double* bary,
                 const int* gate, void* ws, size_t ws_bytes, fcb_stream_t stream);

/* cost of a solved problem: ASYM f.row_sums + sum(g)/m (sinkhorn.py:289),
 * SYM 2 p.row_sums (sinkhorn.py:315).  out: device double. */
FCB_API int fcb_ot_cost(int mode, const double* f, const double* row_sums, int n, const double* g, int m,
                double* out, fcb_stream_t stream);

/* SinkhornSolution.plan (sinkhorn.py:253-256): out (n*m) = exp((f+g-C)/w). */
FCB_API int fcb_ot_plan(const double* X, int n, const double* Y, int m, int d, const double* f,
                const double* g, const double* scal, double* out, fcb_stream_t stream);

/* sinkhorn_flow (sinkhorn.py:338-400): omega, cross + self solves, FlowError
 * test and the envelope gradient, with the warm state (warm_f, warm_p; n
 * each, device, updated in place when warm_valid[0] says so).
 *   flow      : (n*d) out
 *   fstat     : device double[8] = {worst_err, converged, flow_error(0/1),
 *               mean_magnitude, omega, iters_cross, iters_self, 0}
 *   warm_valid: device int[2] {f valid, p valid}; read and set.  NULL = cold.
 *   plan_state/iteration/flow_log/conv_tol (nullable): planner hooks --
 *               a FlowError marks plan_state failed (stage 2); otherwise
 *               flow_log[4*iteration..] = {mean magnitude, inner iterations
 *               of the cross solve, of the self solve, marginal error} and
 *               the convergence test of optimizer.py:251-255 is applied. */
FCB_API size_t fcb_sinkhorn_flow_workspace_bytes(int precision, int n, int m, int d);
FCB_API int fcb_sinkhorn_flow(int precision, const double* X, int n, const double* Y, int m, int d,
                      double omega_fixed, int max_iters, double tol, double* warm_f,
                      double* warm_p, int* warm_valid, double* flow, double* fstat,
                      int* plan_state, int iteration, double* flow_log, double conv_tol,
                      void* ws, size_t ws_bytes, fcb_stream_t stream);

/* sinkhorn_divergence (sinkhorn.py:319-335); out: device double[4] =
 * {divergence, cross cost, self_x cost, self_y cost}. */
FCB_API size_t fcb_sinkhorn_divergence_workspace_bytes(int precision, int n, int m, int d);
FCB_API int fcb_sinkhorn_divergence(int precision, const double* X, int n, const double* Y, int m, int d,
                            double omega_fixed, int max_iters, double tol, double* out,
                            const int* gate, void* ws, size_t ws_bytes, fcb_stream_t stream);
/* The same with the OT(Y, Y) self term cached across calls:
 * Y must be the same point set on every call that shares yy_cache (a device
 * double[5], zeroed = empty: {valid, omega, cost, m, hits}); the M x M self
 * solve is skipped when omega (fixed by omega_fixed, or resolved equal) and m
 * match the cached entry.  Results are bit-identical to the uncached call. */
FCB_API int fcb_sinkhorn_divergence_cached(int precision, const double* X, int n, const double* Y,
                                   int m, int d, double omega_fixed, int max_iters, double tol,
                                   double* out, const int* gate, double* yy_cache, void* ws,
                                   size_t ws_bytes, fcb_stream_t stream);

/* ---- reference density (reference.py) ---------------------------------- */

/* GaussianMixture score / log_density (reference.py:77-110).
 * params (device double): [log_w(k) | log_norm(k) | means(k*d) | chol(k*d*d)]
 * with chol the lower Cholesky factors.  score / logdens nullable. */
FCB_API int fcb_gmm_eval(const double* X, int n, int d, int k, const double* params, double* score,
                 double* logdens, const int* gate, fcb_stream_t stream);

/* SamplePoints.sample (reference.py:140-146) on a device-resident cloud:
 * out (n*d) = src rows idx[0..n) (host-drawn PCG64 indices, int32, uploaded);
 * status (nullable device int): -1, or the first position with an index
 * outside [0, m). */
FCB_API int fcb_gather_rows(const double* src, int m, int d, const int* idx, int n, double* out,
                            int* status, fcb_stream_t stream);

/* ---- Stein variational flow (stein.py) ---------------------------------- */

/* median_bandwidth (stein.py:66-76): exact np.median over all n^2 pairwise
 * distances (diagonal included) by radix selection, then
 * h = med^2 / log_np1 (log_np1 = log(n+1) computed by the caller).
 * hstat: device double[4] = {h, med, clamped, 0}; the BANDWIDTH_FLOOR clamp
 * of stein.py:101-103 is applied. */
FCB_API size_t fcb_median_workspace_bytes(int n);
FCB_API int fcb_median_bandwidth(const double* X, int n, int d, double log_np1, double* hstat,
                         const int* gate, void* ws, size_t ws_bytes, fcb_stream_t stream);

/* stein_flow (stein.py:79-122): out (n*d).  hstat[0] is the (clamped)
 * bandwidth; fixed bandwidths are written there by the caller. */
FCB_API size_t fcb_stein_workspace_bytes(int precision, int n, int d);
FCB_API int fcb_stein_flow(int precision, const double* X, int n, int d, const double* scores,
                   const double* hstat, double* out, const int* gate, void* ws,
                   size_t ws_bytes, fcb_stream_t stream);

/* stein_flow_on_trajectory for the planner: median/fixed bandwidth, GMM
 * score and the flow, plus the mean-magnitude / convergence hooks of
 * fcb_sinkhorn_flow (flow_log row: {mean magnitude, bandwidth, clamped,
 * median}).  fstat as for fcb_sinkhorn_flow with fstat[4] = bandwidth and
 * fstat[5] = clamped. */
FCB_API size_t fcb_stein_flow_full_workspace_bytes(int precision, int n, int d);
FCB_API int fcb_stein_flow_full(int precision, const double* X, int n, int d, int k,
                        const double* gmm_params, double bandwidth_fixed, double log_np1,
                        double* flow, double* fstat, int* plan_state, int iteration,
                        double* flow_log, double conv_tol, void* ws, size_t ws_bytes,
                        fcb_stream_t stream);

/* ---- dynamics and LQR (dynamics.py, lqr.py) ----------------------------- */

/* rollout (dynamics.py:276-312): RK4, zero-order hold.  S (T+1)*ns out,
 * X (T*d, nullable) receives the workspace projection of S[1:]
 * (project_states, dynamics.py:67-69; P is d*ns, device).
 * status: device int; -1 on success, else the step index k+1 of the first
 * non-finite state (RolloutDivergenceError.step).  plan_state/iteration:
 * nullable planner hooks (stage 1). model_params: LTI [A(ns*ns) | B(ns*m)].
 * method 0: sequential RK4, bit-identical to the reference for polynomial
 * models.  method 1: for linear models (single/double integrator, LTI) the
 * RK4 step is the exact affine map s' = Phi s + Gam u and the trajectory is
 * a parallel prefix scan (agrees to rounding); needs a workspace of
 * fcb_rollout_workspace_bytes(ns, T) bytes; nonlinear models run method 0. */
FCB_API size_t fcb_rollout_workspace_bytes(int ns, int T);
FCB_API int fcb_rollout(int model, int ns, int m, const double* model_params, const double* s0,
                const double* U, int T, double dt, double* S, int d, const double* P,
                double* X, int* status, int* plan_state, int iteration, int method,
                double* ws, fcb_stream_t stream);

/* linearize_along (dynamics.py:315-329): A (T*ns*ns), B (T*ns*m). */
FCB_API int fcb_linearize(int model, int ns, int m, const double* model_params, const double* S,
                  const double* U, int T, double* A, double* B, fcb_stream_t stream);

/* solve_flow_lqr (lqr.py:154-200) on explicit A, B (T, ns, ns/m).
 * a: (T*ns) state-space flow.  v (T*m), z ((T+1)*ns), K (T*m*ns), dff (T*m)
 * out (K/dff nullable).  scal: device double[2] = {cost, 0};
 * status: device int, -1 or the time index of a non-finite value. */
FCB_API int fcb_lqr_solve(int ns, int m, int T, double dt, const double* A, const double* B,
                  const double* Q, const double* R, const double* a, double* v, double* z,
                  double* K, double* dff, double* scal, int* status, double* ws,
                  fcb_stream_t stream);
FCB_API size_t fcb_lqr_workspace_bytes(int ns, int m, int T);

/* One planner update (optimizer.py:259-268): linearize along (S, U) on the
 * fly, lift the workspace flow (lqr.py:140-142), solve the flow LQR and
 * write U_next = clamp(U + eta * v*).  lqr_costs[iteration] gets the cost;
 * a Riccati blow-up marks plan_state failed (stage 3).  clamp nullable.
 * The LQR runs in two phases (csrc/lqr_split.cuh): a flow-independent
 * Riccati scan (gains, closed-loop maps) and a per-flow affine phase.
 * mode 0 runs both; mode 1 runs only the affine phase and reuses the Riccati
 * outputs left in `ws` by an earlier mode-0 call -- valid when the model's
 * Jacobians are state-independent (single/double integrator, LTI), whose
 * Riccati inputs are then bitwise identical. */
FCB_API int fcb_plan_update(int model, int ns, int m, const double* model_params, const double* S,
                    const double* U, int T, double dt, int d, const double* P,
                    const double* flow, const double* Q, const double* R, double eta,
                    const double* clamp, double* U_next, double* lqr_costs, int* plan_state,
                    int iteration, int mode, double* ws, size_t ws_bytes, fcb_stream_t stream);
FCB_API size_t fcb_plan_update_workspace_bytes(int ns, int m, int T);

/* The coverage loop of optimizer.py:221-269 for iterations it0..maxit-1 in ONE
 * persistent launch (rollout -> Sinkhorn flow -> LQR affine phase -> control
 * update, device-side stop tests), for the built-in linear models (single /
 * double integrator) with the fp32 resident flow (point sets on chip) and no
 * in-loop metric.  Replaces the per-iteration fcb_rollout / fcb_sinkhorn_flow /
 * fcb_plan_update sequence of the planner (optimizer.py:221-269); results
 * follow the same semantics (warm state, flow_log rows, lqr_costs, plan_state
 * stop codes).  U0/U1 and S0/S1: controls and states of even / odd iterations
 * (iteration it reads U_{it&1}, writes U_{(it+1)&1}).  upd_ws: the
 * fcb_plan_update workspace after a mode-0 call (stored Riccati phase).
 * batch > 1: independent problems of the same shape, one CTA each (inputs
 * stacked per problem: s0, U, S, X, flow, Y, warm state, fstat [8], plan_state
 * [8], flow_log [4*maxit], lqr_costs [maxit], phase_ns [3]); batch 1 spreads
 * the problem over every SM.  Returns FCB_ENOTSUP when the shape/model is not
 * covered (the caller keeps the per-iteration path). */
FCB_API size_t fcb_plan_fused_workspace_bytes(int batch, int T, int M, int d, int m);
FCB_API int fcb_plan_fused(int model, int ns, int m, const double* model_params, const double* s0,
                   double* U0, double* U1, double* S0, double* S1, int T, double dt, int d,
                   const double* P, double* X, double* flow, const double* Q, const double* R,
                   double eta, const double* clamp, const double* Y, int M, double omega_fixed,
                   int max_iters, double tol, double conv_tol, double* warm_f, double* warm_p,
                   int* warm_valid, double* fstat, int* plan_state, double* flow_log,
                   double* lqr_costs, unsigned long long* phase_ns, int it0, int maxit,
                   int batch, const void* upd_ws, void* ws, size_t ws_bytes,
                   fcb_stream_t stream);

/* The same persistent loop with the SVGD flow (stein.py:66-122): per iteration
 * the rollout, the mixture score of every point, the exact median bandwidth
 * (or bandwidth_fixed > 0), the fp64 Stein flow, the LQR affine phase and the
 * control update in one cooperative launch over every SM, for the built-in
 * linear models with a planar workspace and no in-loop metric (T up to 64
 * points per SM).  gmm_params: fcb_gmm_eval's layout with k components;
 * log_np1 = log(T + 1).  flow_log rows, fstat and plan_state as
 * fcb_stein_flow_full + fcb_plan_update.  FCB_ENOTSUP: not covered (the
 * caller keeps the per-iteration path). */
FCB_API size_t fcb_plan_fused_stein_workspace_bytes(int T, int d, int m);
FCB_API int fcb_plan_fused_stein(int model, int ns, int m, const double* model_params,
                         const double* s0, double* U0, double* U1, double* S0, double* S1,
                         int T, double dt, int d, const double* P, double* X, double* flow,
                         const double* Q, const double* R, double eta, const double* clamp,
                         int k, const double* gmm_params, double bandwidth_fixed, double log_np1,
                         double conv_tol, double* fstat, int* plan_state, double* flow_log,
                         double* lqr_costs, unsigned long long* phase_ns, int it0, int maxit,
                         const void* upd_ws, void* ws, size_t ws_bytes, fcb_stream_t stream);

/* ---- M-sharded flows (one process per GPU; distributed.py) ---------------
 * Replaces the row-chunked thread pool of parallel.py:47-66 (used by
 * sinkhorn.py:151-167 and stein.py:110-121) with a split of the reference
 * samples (Sinkhorn) or the SVGD sources across GPUs.  These are the device
 * steps; the caller runs the NCCL collectives between them on the same stream
 * (csrc/shard.cu has the schedule).  ctl: device int[8] loop-control words,
 * eslot: device unsigned long long[2]; both owned by the caller and reset by
 * fcb_shard_init.  Kernels of a finished solve are no-ops. */

/* out = {sum of coordinates (d), sum |p|^2, n}: the per-shard statistics of
 * resolve_omega (sinkhorn.py:136-148), summed over ranks by the caller. */
FCB_API int fcb_point_sums(const double* P, int n, int d, double* out, fcb_stream_t stream);

/* One _lse_rows sweep (sinkhorn.py:151-167) of rows R (nr) against columns S
 * (ns) with column potential pot: L_i = LSE_j((pot_j - |r_i - s_j|^2)/omega).
 * out (nullable) = out_scale omega (out_shift - L) when out_scale != 0, else
 * L (omega = scal[0]: the g-update w (log b - L) is out_scale 1, shift log b);
 * bary (nullable, nr*(d+1)) = {L_i, softmax-weighted mean of the columns}.
 * row_est (nullable, nr): a potential of the rows whose fixed-point relation
 * L_i = row_logw - row_est_i / omega shifts each row's terms near 1 (the fp32
 * fast path needs it; without it the first pass runs the careful loop). */
FCB_API size_t fcb_lse_sweep_workspace_bytes(int precision, int nr, int ns, int d);
FCB_API int fcb_lse_sweep(int precision, const double* R, int nr, const double* S, int ns, int d,
                          const double* scal, const double* pot, const double* row_est,
                          double row_logw, double out_scale, double out_shift, double* out,
                          double* bary, const int* gate, void* ws, size_t ws_bytes,
                          fcb_stream_t stream);

/* Flow start: omega from X and the global Y sums ysum (d+2), both centrings
 * (scal_x: cross solve, scal_s: self solve; resolve_omega layout), f/p from
 * the warm state or zero, ctl/eslot reset.  plan_state != 0 skips the flow. */
FCB_API int fcb_shard_init(int precision, const double* X, int n, int d, const double* ysum,
                           double omega_fixed, const double* warm_f, const double* warm_p,
                           const int* warm_valid, double* scal_x, double* scal_s, double* f,
                           double* p, int* ctl, unsigned long long* eslot, const int* plan_state,
                           fcb_stream_t stream);

/* Cross solve f-update (sinkhorn.py:190-205) from the gathered shard partials
 * gathered[R][n][d+1] = {L_r, barycentre_r}: fixed-order LSE merge, f_new,
 * err, row sums / plan mass / barycentres of the current f, stop decision
 * (stat = {err, iters, converged, 0}); f <- f_new unless stopped. */
FCB_API int fcb_shard_cross_merge(int n, int d, int R, const double* gathered, const double* scal,
                                  double tol, int max_iters, double* f, double* fnext, double* rs,
                                  double* mass, double* ybar, int* ctl, unsigned long long* eslot,
                                  double* stat, fcb_stream_t stream);

/* Self solve (sinkhorn.py:208-236), rows [row0, row0+nown) of X: Lb from
 * fcb_lse_sweep (bary form) -> send[nown][d+4] = {p_new, rho, mass, err_i, xbar}. */
FCB_API int fcb_shard_self_rows(int n, int d, int row0, int nown, const double* Lb,
                                const double* scal, const double* p, double* send, const int* ctl,
                                fcb_stream_t stream);
/* gathered[R][chunk][d+4] (balanced contiguous shards) -> p_new, rho, mass,
 * xbar for all rows, err and the stop decision; p <- p_new unless stopped. */
FCB_API int fcb_shard_self_commit(int n, int d, int R, int chunk, const double* gathered,
                                  double tol, int max_iters, double* p, double* pnext, double* rho,
                                  double* massp, double* xbar, int* ctl, unsigned long long* eslot,
                                  double* stat, fcb_stream_t stream);

/* Envelope gradient (sinkhorn.py:383-391), FlowError test (:370-373), warm
 * state (:393-395) and the planner hooks of fcb_sinkhorn_flow. */
FCB_API size_t fcb_shard_finish_workspace_bytes(int n);
FCB_API int fcb_shard_flow_finish(const double* X, int n, int d, const double* rs,
                                  const double* mass, const double* ybar, const double* rho,
                                  const double* massp, const double* xbar, const double* stat_x,
                                  const double* stat_p, double tol, const double* f,
                                  const double* p, double* warm_f, double* warm_p, int* warm_valid,
                                  double* flow, double* fstat, const double* scal, int* plan_state,
                                  int iteration, double* flow_log, double conv_tol, int* ctl,
                                  void* ws, size_t ws_bytes, fcb_stream_t stream);

/* SVGD (stein.py:79-122) over the source points [col0, col0+ncols) for all n
 * queries: part[n][d+1] = {sum_j k_ij, sum_j k_ij (s_j - (2/h) x'_j)} with x'
 * centred on X[0].  fcb_stein_combine sums R such partials in rank order,
 * writes the flow and runs the planner hooks of fcb_stein_flow_full. */
FCB_API size_t fcb_stein_partial_workspace_bytes(int precision, int n, int nc, int d);
FCB_API int fcb_stein_partial(int precision, const double* X, int n, int d, int col0, int ncols,
                              const double* scores, const double* hstat, double* part,
                              const int* gate, void* ws, size_t ws_bytes, fcb_stream_t stream);
/* median_bandwidth (stein.py:66-76) with the pair tiles split across ranks:
 * init; then for pass = 0..5: fcb_median_shard_pass over this rank's tiles
 * [tile_lo, tile_hi) of the fcb_median_tiles(n) upper-triangle tiles, an
 * all_reduce(SUM) of the 2 x 2048 uint64 histogram at byte offset
 * fcb_median_hist_offset() of ws, fcb_median_shard_select (every rank picks
 * the same digit); then fcb_median_shard_finish writes hstat as
 * fcb_median_bandwidth does.  ws: fcb_median_workspace_bytes(n). */
FCB_API long long fcb_median_tiles(int n);
FCB_API size_t fcb_median_hist_offset(void);
FCB_API int fcb_median_shard_init(int n, void* ws, size_t ws_bytes, const int* gate,
                                  fcb_stream_t stream);
FCB_API int fcb_median_shard_pass(const double* X, int n, int d, int pass, long long tile_lo,
                                  long long tile_hi, void* ws, const int* gate,
                                  fcb_stream_t stream);
FCB_API int fcb_median_shard_select(int n, int pass, void* ws, const int* gate,
                                    fcb_stream_t stream);
FCB_API int fcb_median_shard_finish(int n, double log_np1, double* hstat, void* ws,
                                    const int* gate, fcb_stream_t stream);
FCB_API size_t fcb_stein_combine_workspace_bytes(int n);
FCB_API int fcb_stein_combine(const double* X, int n, int d, int R, const double* parts,
                              const double* hstat, double* flow, double* fstat, int* plan_state,
                              int iteration, double* flow_log, double conv_tol, void* ws,
                              size_t ws_bytes, fcb_stream_t stream);

/* ---- TSP-waypoint baseline (tsp.py) ---------------------------------------
 * build_tour (tsp.py:120-147) for `batch` independent point sets of n points
 * (points: batch*n*d, row-major per problem), one CTA each: nearest-neighbour
 * order from starts[b] (drawn on the host from stream [seed, 4]) refined by
 * first-improving 2-opt moves (tsp.py:92-117) until none improves or `budget`
 * moves were made.  order: batch*n out (int32); moves: batch out (nullable).
 * Same arithmetic as the reference, so the orders are identical. */
FCB_API int fcb_tsp_tours(const double* points, int batch, int n, int d, const int* starts,
                          int budget, int* order, int* moves, fcb_stream_t stream);

/* ---- measurement helpers ------------------------------------------------- */

/* MUFU.EX2 / FFMA throughput probe used by bench.py for the roofline
 * denominators.  out: device double[2] = {ex2 ops, ffma ops} performed;
 * the caller times the launch with events. */
FCB_API int fcb_peak_probe(int which, int iters, double* out, fcb_stream_t stream);

/* Debug builds (-DFCB_TIMELINE): globaltimer stamps of block 0 at every grid
 * barrier of the persistent solvers, copied to a HOST array; returns the
 * count and resets the log.  Production builds return 0. */
FCB_API int fcb_debug_timeline(unsigned long long* host_out, int cap);

/* Work items of the chunked solver that fell back from the fp32 fast path to
 * the careful loop since the last call (synchronises the device; resets). */
FCB_API long long fcb_debug_careful_items(void);

/* Rows of the resident flow kernel (rs_flow_kernel) whose fp32 streaming pass
 * was refused and redone by the careful pass since the last call
 * (synchronises the device; resets). */
FCB_API long long fcb_debug_careful_rows_resident(void);

#ifdef __cplusplus
}
#endif

#endif /* FLOWCOVER_B200_H */
