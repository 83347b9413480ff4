"""GSC-Falkon / LogFalkon CPU oracle (Appendix B, Alg. 2 of arXiv 2006.10350) — plain,
slow, fp64.  TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / --impl reference legs may import it; the CUDA path never does.

It follows Alg. 2 function by function, in the paper's order, with the
readings g1-g7 of DESIGN.md §3 where the pseudocode is garbled or silent:

  g1  LinOp's D is the curvature at the CURRENT Newton iterate alpha_0 (PAPER.md:1051-1053:
      "D_k ... l''(f_k(x_i), y_i)"), not at the CG direction beta (PAPER.md:981 computes
      z from beta, which would make LinOp non-linear).
  g2  RHS: Alg. 2 writes k(X, X_m) y; the Newton system of PAPER.md:1051-1053 for
      the NEW iterate is  (Knm^T D Knm + mu n K) alpha = Knm^T (D z - g),  g_i = l'(z_i, y_i),
      z = Knm alpha_0, which is Knm^T y for the squared loss (the Falkon case).  So the
      working response D z - g replaces y.
  g3  Regularisation mu n (Alg. 1's lambda n convention), not the appendix's mu; D = I makes
      the step exactly Alg. 1 (tested).
  g4  "CG solver starting from alpha_0" = CG on beta from beta_0 = A T alpha_0
      (the inverse of alpha = T^-1 A^-1 beta).
  g5  The outer loop: the levels mu_k and CG iterations are an explicit
      path (mus, iters); `newton_path` builds Alg. 2's geometric path mu_{k+1} = q mu_k,
      stopping when mu_{k+1} < lambda, then one final step at lambda with T iterations.
      "alpha_last <- alpha_k" is read as the latest iterate.
  g6  K = Kmm + delta I (the jitter of reading c6) in the regulariser, as in Alg. 1.
  g7  Losses: logistic l(z, y) = log(1 + exp(-y z)), y in {-1, +1} (Example 1(a),
      PAPER.md:1026); squared l = (z - y)^2 / 2 (the reduction to Falkon).

Pins (tests/test_gsc_oracle.py): loss values/derivatives (finite
differences), squared loss == oracle.fit (Alg. 1), first logistic step from 0 ==
oracle.fit(2y, 4 mu) (D = I/4), t >= m step == the dense Newton step, repeated steps converge
to the minimiser found by scipy.optimize, label negation, weighted preconditioner factor
identities, objective decrease along the path.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla

from .falkon_oracle import DEFAULT_JITTER, NonFinite, NotPositiveDefinite, kmm, knm_t_vec, knm_vec

__all__ = ["LOGISTIC", "SQUARED", "loss_eval", "weighted_preconditioner", "weighted_linop",
           "weighted_falkon", "gsc_falkon", "newton_path", "objective", "cg_from"]

LOGISTIC = 0
SQUARED = 1


def loss_eval(kind: int, z, y):
    """(l, l', l'') of the loss in its first argument (Def. 1, Example 1(a)); numerically
    stable forms (softplus) so |z| large does not overflow."""
    z = np.asarray(z, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if kind == LOGISTIC:
        s = y * z
        val = np.logaddexp(0.0, -s)                      # log(1 + e^{-s})
        sig_neg = 0.5 * (1.0 - np.tanh(0.5 * s))         # sigma(-s) = 1 / (1 + e^{s})
        d1 = -y * sig_neg
        d2 = sig_neg * (1.0 - sig_neg)                   # sigma(s) sigma(-s)  (y^2 = 1)
        return val, d1, d2
    if kind == SQUARED:
        r = z - y
        return 0.5 * r * r, r, np.ones_like(r)
    raise ValueError(f"unknown loss {kind}")


def weighted_preconditioner(C, yC, alpha, loss: int, kernel: int, sigma: float, mu: float,
                            jitter: float = DEFAULT_JITTER):
    """Alg. 2 WeightedPreconditioner, in its order:
        K_mm = k(X_m, X_m)                         (line 1)
        z = K_mm alpha                             (line 2, predictions on the Nystrom points)
        T = chol(K_mm + delta I)                   (line 3; reading g6 / c6)
        D = diag(l''(z_j, y_j))                    (line 4)
        M = (1/m) T D T^T + mu I                   (line 5)
        A = chol(M)                                (line 6)
    Returns (T, A, z), T and A upper with T^T T = K_mm + delta I, A^T A = M."""
    K = kmm(C, kernel, sigma)
    m = K.shape[0]
    z = K @ np.asarray(alpha, dtype=np.float64)
    try:
        T = sla.cholesky(K + jitter * np.eye(m), lower=False)
    except np.linalg.LinAlgError:
        raise NotPositiveDefinite(0) from None
    _, _, Dm = loss_eval(loss, z, yC)
    M = (T * Dm[None, :]) @ T.T / m + mu * np.eye(m)
    try:
        A = sla.cholesky(M, lower=False)
    except np.linalg.LinAlgError:
        raise NotPositiveDefinite(1) from None
    return T, A, z


def _su(U, b, trans):
    return sla.solve_triangular(U, b, lower=False, trans="T" if trans else "N")


def weighted_linop(beta, X, C, T, A, D, mu: float, kernel: int, sigma: float, n_global=None):
    """Alg. 2 WeightedFalkon.LinOp, D fixed at the current iterate
    (reading g1), read as Eq. (9) (reading c1):
        v = A^-1 beta;  c = Knm^T D Knm T^-1 v;  return A^-T (T^-T c + mu n v)."""
    n = X.shape[0] if n_global is None else n_global
    v = _su(A, beta, False)
    w = knm_vec(X, C, _su(T, v, False), kernel, sigma)
    c = knm_t_vec(X, C, D * w, kernel, sigma)
    return _su(A, _su(T, c, True) + mu * n * v, True)


def cg_from(op, b, x0, t: int):
    """Textbook CG from x0 (reading g4): r = b - op(x0), then exactly t iterations with the
    breakdown rules of reading c9.  Returns (x, iterations_run)."""
    x = np.array(x0, dtype=np.float64, copy=True)
    r = np.asarray(b, dtype=np.float64) - op(x)
    p = r.copy()
    rho = float(r @ r)
    it = 0
    for k in range(1, t + 1):
        if rho == 0.0:
            break
        q = op(p)
        gamma = float(p @ q)
        if not (gamma > 0.0) or not math.isfinite(gamma):
            raise NonFinite(k)
        a = rho / gamma
        x = x + a * p
        r = r - a * q
        rho_new = float(r @ r)
        if not math.isfinite(rho_new):
            raise NonFinite(k)
        p = r + (rho_new / rho) * p
        rho = rho_new
        it = k
    return x, it


def weighted_falkon(X, y, C, yC, loss: int, kernel: int, sigma: float, mu: float, t: int,
                    alpha0, jitter: float = DEFAULT_JITTER):
    """Alg. 2 WeightedFalkon: one approximate Newton step at level mu.
        T, A = WeightedPreconditioner(X_m, y_m, alpha0, mu)             (line 2)
        z = Knm alpha0; D = diag(l''(z, y)); g = l'(z, y)               (readings g1, g2)
        R = A^-T T^-T Knm^T (D z - g)                                   (line 9, reading g2)
        beta = CG(LinOp, R, t) from beta_0 = A T alpha0                 (line 10, reading g4)
        return T^-1 A^-1 beta                                           (line 11)"""
    X = np.asarray(X, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    alpha0 = np.asarray(alpha0, dtype=np.float64)
    T, A, _ = weighted_preconditioner(C, yC, alpha0, loss, kernel, sigma, mu, jitter)
    z = knm_vec(X, C, alpha0, kernel, sigma)
    _, g, D = loss_eval(loss, z, y)
    R = _su(A, _su(T, knm_t_vec(X, C, D * z - g, kernel, sigma), True), True)
    beta0 = A @ (T @ alpha0)
    beta, _ = cg_from(lambda b: weighted_linop(b, X, C, T, A, D, mu, kernel, sigma), R, beta0, t)
    return _su(T, _su(A, beta, False), False)


def newton_path(mu0: float, q: float, lam: float, t: int, t_final: int):
    """Alg. 2 GSC-Falkon's level schedule (reading g5): mu_0, q mu_0, ...
    while mu_k >= lam (the step at mu_k runs, then mu_{k+1} = q mu_k; stop when mu_{k+1} <
    lam), then one final WeightedFalkon at lam with t_final iterations."""
    if not (mu0 > 0 and 0 < q < 1 and lam > 0):
        raise ValueError("need mu0 > 0, 0 < q < 1, lam > 0")
    mus, its = [], []
    mu = mu0
    while True:
        mus.append(mu)
        its.append(t)
        mu = q * mu
        if mu < lam:
            break
    mus.append(lam)
    its.append(t_final)
    return mus, its


def gsc_falkon(X, y, C, yC, loss: int, kernel: int, sigma: float, mus, iters,
               jitter: float = DEFAULT_JITTER, return_path: bool = False):
    """Alg. 2 GSC-Falkon: alpha_0 = 0, then alpha <- WeightedFalkon(mu_k,
    t_k, alpha) along the path (reading g5).  C, yC = the Nystrom points and their labels
    (sampled by the caller, reading c11)."""
    alpha = np.zeros(np.asarray(C).shape[0], dtype=np.float64)
    path = []
    for mu, t in zip(mus, iters):
        alpha = weighted_falkon(X, y, C, yC, loss, kernel, sigma, float(mu), int(t), alpha, jitter)
        path.append(alpha.copy())
    return (alpha, path) if return_path else alpha


def objective(X, y, C, alpha, loss: int, kernel: int, sigma: float, mu: float,
              jitter: float = DEFAULT_JITTER):
    """J(alpha) = (1/n) sum_i l(f(x_i), y_i) + (mu/2) alpha^T (K_mm + delta I) alpha: the
    regularised empirical risk of Eq. (2) restricted to the Nystrom model of Eq. (4), whose
    Newton system the weighted step solves (readings g2, g3, g6)."""
    z = knm_vec(X, C, alpha, kernel, sigma)
    val, _, _ = loss_eval(loss, z, y)
    K = kmm(C, kernel, sigma) + jitter * np.eye(len(alpha))
    return float(np.mean(val) + 0.5 * mu * alpha @ (K @ alpha))

