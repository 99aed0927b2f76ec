"""CPU oracle for the flowcover hot path -- TEST INFRASTRUCTURE ONLY.

A float64 numpy restatement of the reference algorithms in
/root/reference/pkg/src/flowcover (stein.py, sinkhorn.py, reference.py,
dynamics.py, lqr.py, optimizer.py).  Every function cites the reference
lines it follows.  It is used by tests/ (as the parity checker), by
__graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
legs (as the timed CPU baseline).  The product path never imports it.

Differences from the reference, none of which change a single output bit:
  * cost matrices are formed per row block from the points instead of being
    materialised whole (the row-block values and per-row reductions are the
    reference's exactly: same elementwise operations, same reduction axis),
    so the oracle also runs at sizes the reference cannot hold;
  * row blocks may be processed by a thread pool (`workers`), the same
    data-parallel scheme as the reference's run_chunked (parallel.py:47-66).

Parity pin: tests/test_oracle_golden.py checks this module against golden
vectors produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.linalg import cho_solve, cholesky

AUTO_OMEGA_FACTOR = 0.05  # sinkhorn.py:65
OMEGA_FLOOR = 1e-12  # sinkhorn.py:66
EXP_CLIP = 500.0  # sinkhorn.py:67
BANDWIDTH_FLOOR = 1e-12  # stein.py:34
LOG_2PI = float(np.log(2.0 * np.pi))


# ---------------------------------------------------------------------------
# execution helper (parallel.py:38-66)
# ---------------------------------------------------------------------------
def _blocks(total: int, chunk: int):
    return [(lo, min(lo + chunk, total)) for lo in range(0, total, chunk)]


def _for_blocks(fn, total: int, chunk: int, workers: int) -> None:
    spans = _blocks(total, chunk)
    if workers <= 1 or len(spans) <= 1:
        for lo, hi in spans:
            fn(lo, hi)
        return
    with ThreadPoolExecutor(max_workers=workers) as pool:
        list(pool.map(lambda s: fn(*s), spans))


# ---------------------------------------------------------------------------
# distances (stein.py:57-63, sinkhorn.py:127-133)
# ---------------------------------------------------------------------------
def sqdist(P: np.ndarray, Q: np.ndarray) -> np.ndarray:
    """|p_i - q_j|^2 accumulated coordinate by coordinate, first coordinate first."""
    out = np.square(P[:, :1] - Q[:, 0][None, :])
    for k in range(1, P.shape[1]):
        out += np.square(P[:, k : k + 1] - Q[:, k][None, :])
    return out


# ---------------------------------------------------------------------------
# entropic OT (sinkhorn.py:136-400)
# ---------------------------------------------------------------------------
def resolve_omega(omega, X: np.ndarray, Y: np.ndarray) -> float:
    """sinkhorn.py:136-148: 0.05 * (mean|x|^2 + mean|y|^2 - 2 <xbar, ybar>), floored."""
    if not isinstance(omega, str):
        return float(omega)
    xbar, ybar = X.mean(axis=0), Y.mean(axis=0)
    msq = float((X * X).sum(axis=1).mean() + (Y * Y).sum(axis=1).mean() - 2.0 * xbar @ ybar)
    return max(AUTO_OMEGA_FACTOR * msq, OMEGA_FLOOR)


def lse_sweep(R: np.ndarray, S: np.ndarray, pot: np.ndarray, omega: float,
              chunk: int = 256, workers: int = 1) -> np.ndarray:
    """out_i = LSE_j((pot_j - |r_i - s_j|^2) / omega) (sinkhorn.py:151-167).

    The cost block of rows [lo, hi) is formed on the fly; per-row reductions
    run along the contiguous axis exactly as in the reference.
    """
    out = np.empty(R.shape[0])

    def block(lo: int, hi: int) -> None:
        z = (pot[None, :] - sqdist(R[lo:hi], S)) / omega
        top = z.max(axis=1)
        np.exp(z - top[:, None], out=z)
        out[lo:hi] = top + np.log(z.sum(axis=1))

    _for_blocks(block, R.shape[0], chunk, workers)
    return out


def solve_asymmetric(X, Y, omega, max_iters, tol, f0=None, chunk=256, workers=1, log=None):
    """Alternating dual updates (sinkhorn.py:170-205).

    Returns (f, g, row_sums, err, iters, converged) with f the pre-update
    potential the error was measured on.
    """
    n, m = X.shape[0], Y.shape[0]
    log_a, log_b = -math.log(n), -math.log(m)
    f = np.zeros(n) if f0 is None else np.array(f0, dtype=np.float64)
    it = 0
    while True:
        it += 1
        g = omega * (log_b - lse_sweep(Y, X, f, omega, chunk, workers))
        f_next = omega * (log_a - lse_sweep(X, Y, g, omega, chunk, workers))
        delta = np.minimum((f - f_next) / omega, EXP_CLIP)
        err = float(np.abs(np.expm1(delta)).max() / n)
        if log is not None:
            log.append(("asym", it, err))
        if err <= tol or it >= max_iters:
            return f, g, np.exp(delta + log_a), err, it, err <= tol
        f = f_next


def solve_symmetric(X, omega, max_iters, tol, p0=None, chunk=256, workers=1):
    """Damped self-transport fixed point (sinkhorn.py:208-236)."""
    n = X.shape[0]
    log_a = -math.log(n)
    p = np.zeros(n) if p0 is None else np.array(p0, dtype=np.float64)
    it = 0
    while True:
        it += 1
        target = omega * (log_a - lse_sweep(X, X, p, omega, chunk, workers))
        delta = np.minimum((p - target) / omega, EXP_CLIP)
        err = float(np.abs(np.expm1(delta)).max() / n)
        if err <= tol or it >= max_iters:
            return p, np.exp(delta + log_a), err, it, err <= tol
        p = 0.5 * (p + target)


def entropic_ot(X, Y, omega="auto", max_iters=1000, tol=1e-6, f0=None, chunk=256, workers=1):
    """sinkhorn.py:259-300 (cost = f . row_sums + sum(g) / m)."""
    X, Y = np.atleast_2d(X).astype(np.float64), np.atleast_2d(Y).astype(np.float64)
    w = resolve_omega(omega, X, Y)
    f, g, rs, err, iters, conv = solve_asymmetric(X, Y, w, max_iters, tol, f0, chunk, workers)
    cost = float(f @ rs + g.sum() / Y.shape[0])
    return dict(f=f, g=g, row_sums=rs, cost=cost, iters=iters, converged=conv, err=err, omega=w)


def self_cost(X, omega, max_iters, tol, chunk=256, workers=1) -> float:
    """sinkhorn.py:303-316: 2 p . row_sums of the symmetric solve."""
    p, rs, _, _, _ = solve_symmetric(X, omega, max_iters, tol, None, chunk, workers)
    return float(2.0 * (p @ rs))


def sinkhorn_divergence(X, Y, omega="auto", max_iters=1000, tol=1e-6, chunk=256, workers=1):
    """sinkhorn.py:319-335, one omega for all three terms."""
    X, Y = np.atleast_2d(X).astype(np.float64), np.atleast_2d(Y).astype(np.float64)
    w = resolve_omega(omega, X, Y)
    cross = entropic_ot(X, Y, w, max_iters, tol, None, chunk, workers)["cost"]
    return cross - 0.5 * (self_cost(X, w, max_iters, tol, chunk, workers)
                          + self_cost(Y, w, max_iters, tol, chunk, workers))


def plan_weighted_sums(R, S, a, b, omega, chunk=256, workers=1):
    """Row sums of (T_ij * s_j) for T_ij = exp((a_i + b_j - |r_i - s_j|^2)/omega)
    (the plan/gradient products of sinkhorn.py:384-391), per row block."""
    out = np.empty((R.shape[0], S.shape[1]))

    def block(lo, hi):
        T = np.exp((a[lo:hi, None] + b[None, :] - sqdist(R[lo:hi], S)) / omega)
        for k in range(S.shape[1]):
            out[lo:hi, k] = (T * S[:, k][None, :]).sum(axis=1)

    _for_blocks(block, R.shape[0], chunk, workers)
    return out


def sinkhorn_flow(X, Y, omega="auto", max_iters=1000, tol=1e-6, warm=None, chunk=256,
                  workers=1, stats=None):
    """Minus the divergence gradient (sinkhorn.py:338-400).

    warm: dict with optional 'f'/'p' (updated in place like SinkhornWarmState).
    Raises RuntimeError('FlowError ...') when a marginal error exceeds 100 tol.
    """
    X, Y = np.atleast_2d(X).astype(np.float64), np.atleast_2d(Y).astype(np.float64)
    n = X.shape[0]
    w = resolve_omega(omega, X, Y)
    f0 = warm.get("f") if warm is not None else None
    f0 = f0 if f0 is not None and f0.shape[0] == n else None
    f, g, r, err_x, it_x, conv_x = solve_asymmetric(X, Y, w, max_iters, tol, f0, chunk, workers)
    p0 = warm.get("p") if warm is not None else None
    p0 = p0 if p0 is not None and p0.shape[0] == n else None
    p, rho, err_p, it_p, conv_p = solve_symmetric(X, w, max_iters, tol, p0, chunk, workers)
    worst = max(err_x, err_p)
    if stats is not None:
        stats.update(iters_cross=it_x, iters_self=it_p, omega=w, worst=worst)
    if worst > 100.0 * tol:
        raise RuntimeError(f"FlowError: marginals violated by {worst:.3e}")
    ty = plan_weighted_sums(X, Y, f, g, w, chunk, workers)
    px = plan_weighted_sums(X, X, p, p, w, chunk, workers)
    grad = 2.0 * (r[:, None] * X - ty) - 2.0 * (rho[:, None] * X - px)
    if warm is not None:
        warm["f"], warm["p"] = f, p
    return -grad, conv_x and conv_p, worst


# ---------------------------------------------------------------------------
# Gaussian mixture (reference.py:25-176)
# ---------------------------------------------------------------------------
class Mixture:
    """Cholesky-cached mixture (reference.py:55-67) with score/log density."""

    def __init__(self, weights, means, covariances):
        self.w = np.asarray(weights, dtype=np.float64)
        self.mu = np.asarray(means, dtype=np.float64)
        self.cov = np.asarray(covariances, dtype=np.float64)
        self.L = np.stack([cholesky(c, lower=True) for c in self.cov])
        d = self.mu.shape[1]
        self.log_norm = 0.5 * d * LOG_2PI + np.log(np.diagonal(self.L, axis1=1, axis2=2)).sum(1)

    def _terms(self, X):
        """(log pdf (n, k), pulls (k, n, d)) -- reference.py:77-94."""
        X = np.atleast_2d(X).astype(np.float64)
        k = self.mu.shape[0]
        lp = np.empty((X.shape[0], k))
        pulls = np.empty((k,) + X.shape)
        for c in range(k):
            diff = X - self.mu[c]
            pull = cho_solve((self.L[c], True), diff.T).T
            pulls[c] = pull
            lp[:, c] = -0.5 * np.einsum("nd,nd->n", diff, pull) - self.log_norm[c]
        return lp, pulls

    def log_density(self, X):
        lp, _ = self._terms(X)
        s = lp + np.log(self.w)
        top = s.max(axis=1)
        return top + np.log(np.exp(s - top[:, None]).sum(axis=1))

    def score(self, X):
        """reference.py:103-110: responsibility-weighted negative pulls."""
        lp, pulls = self._terms(X)
        s = lp + np.log(self.w)
        s -= s.max(axis=1, keepdims=True)
        r = np.exp(s)
        r /= r.sum(axis=1, keepdims=True)
        return -np.einsum("nk,knd->nd", r, pulls)

    def sample(self, n, seed):
        """reference.py:112-119 (ancestral draws, numpy PCG64)."""
        rng = np.random.default_rng(seed)
        comp = rng.choice(self.mu.shape[0], size=n, p=self.w)
        z = rng.standard_normal((n, self.mu.shape[1]))
        return self.mu[comp] + np.einsum("nij,nj->ni", self.L[comp], z)


def benchmark_mixture(dim=2) -> Mixture:
    """reference.py:159-176."""
    xy = np.array([(0.25, 0.25), (0.75, 0.35), (0.4, 0.8)])
    means = xy if dim == 2 else np.column_stack([xy, [0.25, 0.75, 0.5]])
    return Mixture(np.full(3, 1.0 / 3.0), means, np.tile(0.02 * np.eye(dim), (3, 1, 1)))


# ---------------------------------------------------------------------------
# Stein flow (stein.py:66-122)
# ---------------------------------------------------------------------------
def median_bandwidth(X) -> float:
    """stein.py:66-76: np.median over all n^2 distances (diagonal included)."""
    X = np.atleast_2d(X).astype(np.float64)
    n = X.shape[0]
    if n == 1:
        return 1.0
    med = float(np.median(np.sqrt(sqdist(X, X))))
    return med * med / math.log(n + 1.0)


def stein_flow(X, q: Mixture, bandwidth="median", chunk=256, workers=1):
    """stein.py:79-122.  Returns (flow, h, clamped)."""
    X = np.atleast_2d(X).astype(np.float64)
    n, d = X.shape
    h = median_bandwidth(X) if bandwidth == "median" else float(bandwidth)
    clamped = h <= BANDWIDTH_FLOOR
    if clamped:
        h = BANDWIDTH_FLOOR
    sc = q.score(X)
    out = np.empty((n, d))

    def block(lo, hi):
        K = np.exp(-sqdist(X[lo:hi], X) / h)
        ks = K.sum(axis=1)
        for k in range(d):
            attract = (K * sc[:, k][None, :]).sum(axis=1)
            pull_in = (K * X[:, k][None, :]).sum(axis=1)
            out[lo:hi, k] = (1.0 / n) * (attract + (2.0 / h) * (X[lo:hi, k] * ks - pull_in))

    _for_blocks(block, n, chunk, workers)
    return out, h, clamped


# ---------------------------------------------------------------------------
# dynamics (dynamics.py:72-329)
# ---------------------------------------------------------------------------
def model_fns(name: str):
    """(f, jac_A, jac_B, P) for the device-supported models (dynamics.py:72-181)."""
    if name == "single_integrator_2d":
        return (lambda s, u: np.asarray(u, dtype=np.float64),
                lambda s, u: np.zeros((2, 2)), lambda s, u: np.eye(2), np.eye(2))
    if name == "diff_drive":
        def f(s, u):
            return np.array([u[0] * np.cos(s[2]), u[0] * np.sin(s[2]), u[1]])

        def ja(s, u):
            A = np.zeros((3, 3))
            A[0, 2], A[1, 2] = -u[0] * np.sin(s[2]), u[0] * np.cos(s[2])
            return A

        def jb(s, u):
            return np.array([[np.cos(s[2]), 0.0], [np.sin(s[2]), 0.0], [0.0, 1.0]])

        return f, ja, jb, np.array([[1.0, 0, 0], [0, 1.0, 0]])
    if name == "aircraft_3d":
        Bc = np.zeros((6, 3))
        Bc[3, 0] = Bc[4, 1] = Bc[5, 2] = 1.0

        def f(s, u):
            cg = np.cos(s[4])
            return np.array([s[5] * cg * np.cos(s[3]), s[5] * cg * np.sin(s[3]),
                             s[5] * np.sin(s[4]), u[0], u[1], u[2]])

        def ja(s, u):
            psi, gam, v = s[3], s[4], s[5]
            A = np.zeros((6, 6))
            A[0, 3:6] = (-v * np.cos(gam) * np.sin(psi), -v * np.sin(gam) * np.cos(psi),
                         np.cos(gam) * np.cos(psi))
            A[1, 3:6] = (v * np.cos(gam) * np.cos(psi), -v * np.sin(gam) * np.sin(psi),
                         np.cos(gam) * np.sin(psi))
            A[2, 4:6] = (v * np.cos(gam), np.sin(gam))
            return A

        P = np.zeros((3, 6))
        P[0, 0] = P[1, 1] = P[2, 2] = 1.0
        return f, ja, (lambda s, u: Bc.copy()), P
    if name == "double_integrator_2d":
        A = np.zeros((4, 4))
        A[0, 2] = A[1, 3] = 1.0
        B = np.zeros((4, 2))
        B[2, 0] = B[3, 1] = 1.0
        P = np.zeros((2, 4))
        P[0, 0] = P[1, 1] = 1.0
        return (lambda s, u: np.array([s[2], s[3], u[0], u[1]]),
                lambda s, u: A.copy(), lambda s, u: B.copy(), P)
    raise ValueError(f"oracle has no model {name!r}")


def rollout(f, s0, U, dt):
    """RK4 with zero-order hold (dynamics.py:276-312); returns (S, fail_step or -1)."""
    U = np.asarray(U, dtype=np.float64)
    T = U.shape[0]
    S = np.empty((T + 1, len(s0)))
    S[0] = s = np.asarray(s0, dtype=np.float64)
    half, sixth = 0.5 * dt, dt / 6.0
    with np.errstate(over="ignore", invalid="ignore"):
        for k in range(T):
            u = U[k]
            k1 = f(s, u)
            k2 = f(s + half * k1, u)
            k3 = f(s + half * k2, u)
            k4 = f(s + dt * k3, u)
            s = s + sixth * (k1 + 2.0 * (k2 + k3) + k4)
            if not np.isfinite(s).all():
                return S, k + 1
            S[k + 1] = s
    return S, -1


def linearize(ja, jb, S, U):
    """dynamics.py:315-329."""
    T = U.shape[0]
    A = np.stack([ja(S[k], U[k]) for k in range(T)])
    B = np.stack([jb(S[k], U[k]) for k in range(T)])
    return A, B


# ---------------------------------------------------------------------------
# flow-matching LQR (lqr.py:154-200)
# ---------------------------------------------------------------------------
def solve_flow_lqr(A, B, dt, a, Q, R):
    """Backward Riccati with affine term, forward z/v/cost.  Returns dict or
    raises ArithmeticError(k) when the sweep leaves the finite range."""
    T, n, _ = A.shape
    m = B.shape[2]
    Qb, Rb = dt * Q, dt * R
    F = np.eye(n)[None] + dt * A
    G = dt * B
    K = np.empty((T, m, n))
    dff = np.empty((T, m))
    P, p = np.zeros((n, n)), np.zeros(n)
    for k in range(T - 1, -1, -1):
        Fk, Gk = F[k], G[k]
        H = Rb + Gk.T @ (P @ Gk)
        rhs = np.concatenate([Gk.T @ (P @ Fk), -(Gk.T @ p)[:, None]], axis=1)
        sol = np.linalg.solve(H, rhs)
        K[k], dff[k] = sol[:, :n], sol[:, n]
        closed = Fk - Gk @ K[k]
        P = Qb + Fk.T @ (P @ closed)
        P = 0.5 * (P + P.T)
        p = -(Qb @ a[k]) + closed.T @ p
        if not (np.isfinite(P).all() and np.isfinite(p).all()):
            raise ArithmeticError(k)
    z = np.zeros((T + 1, n))
    v = np.empty((T, m))
    cost = 0.0
    for k in range(T):
        v[k] = dff[k] - K[k] @ z[k]
        e = a[k] - z[k]
        cost += e @ (Qb @ e) + v[k] @ (Rb @ v[k])
        z[k + 1] = F[k] @ z[k] + G[k] @ v[k]
    return dict(v=v, z=z, K=K, d=dff, cost=float(cost))


# ---------------------------------------------------------------------------
# planner loop (optimizer.py:171-304)
# ---------------------------------------------------------------------------
def plan(model_name, s0, dt, T, method, eta, iterations, *, q=None, targets=None, seed=0,
         conv_tol=0.0, omega="auto", max_iters=1000, tol=1e-6, bandwidth="median",
         q_weight=1.0, r_weight=0.1, clamp=None, init="random_small", init_scale=1e-2,
         workers=1, chunk=256, record=None):
    """The outer loop of optimizer.py:221-269 without the metric cadence.

    Returns dict(S, U, flow_norms, lqr_costs, inner=[(iters_cross, iters_self)],
    converged).  record (list) receives per-iteration (S, flow) if given.
    """
    f, ja, jb, P = model_fns(model_name)
    m = 3 if model_name == "aircraft_3d" else 2
    if init == "zeros":
        U = np.zeros((T, m))
    else:
        rng = np.random.default_rng(np.random.SeedSequence([seed, 1]))
        U = init_scale * rng.standard_normal((T, m))
    if clamp is not None:
        np.clip(U, -np.asarray(clamp), np.asarray(clamp), out=U)
    if method == "sinkhorn" and targets is None:
        targets = q.sample(T, [seed, 2])
    Qw, Rw = q_weight * (P.T @ P), r_weight * np.eye(m)
    warm: dict = {}
    norms, costs, inner = [], [], []
    converged = False
    for _ in range(iterations):
        S, fail = rollout(f, s0, U, dt)
        if fail >= 0:
            raise ArithmeticError(f"rollout diverged at step {fail}")
        X = S[1:] @ P.T
        if method == "sinkhorn":
            stats: dict = {}
            a, _, _ = sinkhorn_flow(X, targets, omega, max_iters, tol, warm, chunk, workers, stats)
            inner.append((stats["iters_cross"], stats["iters_self"]))
        else:
            a, _, _ = stein_flow(X, q, bandwidth, chunk, workers)
        if record is not None:
            record.append((S.copy(), a.copy()))
        norms.append(float(np.sqrt((a * a).sum(axis=1)).mean()))
        if norms[-1] < conv_tol:
            converged = True
            break
        A, B = linearize(ja, jb, S, U)
        sol = solve_flow_lqr(A, B, dt, a @ P, Qw, Rw)
        costs.append(sol["cost"])
        U = U + eta * sol["v"]
        if clamp is not None:
            np.clip(U, -np.asarray(clamp), np.asarray(clamp), out=U)
    S, _ = rollout(f, s0, U, dt)
    return dict(S=S, U=U, flow_norms=np.array(norms), lqr_costs=np.array(costs), inner=inner,
                converged=converged)
