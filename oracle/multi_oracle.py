"""Multi-output Falkon CPU oracle — TEST INFRASTRUCTURE ONLY (same
import rules as falkon_oracle.py).  fp64, written from the paper.

The paper treats a k-class problem (TIMIT, 144 classes) as k outputs of the
same Nystrom model: Eq. (4) with alpha in R^{m x k} and Alg. 1 applied to
each column of Y.  The k CG runs are independent (reading c9 per column) and share the
preconditioner and the kernel matrix; here every step is written in matrix form (one
Knm^T (Knm V) per row block for all columns; CG with per-column scalars).

Pins (tests/test_multi_oracle.py): each column equals the single-output oracle (product,
fit, predict), k = 1 reduces to it, and column permutation commutes with the fit.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .falkon_oracle import (DEFAULT_JITTER, NonFinite, _block_rows, kernel_block,
                            preconditioner)

__all__ = ["knm_t_knm_mat", "fit_multi", "predict_multi"]


def knm_t_knm_mat(X, C, V, kernel: int, sigma: float, block_rows: int | None = None):
    """U = Knm^T (Knm V) = sum_b k(X_b, C)^T (k(X_b, C) V), V in R^{m x k}."""
    X = np.asarray(X, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    q = _block_rows(C.shape[0], block_rows)
    U = np.zeros_like(V)
    for s in range(0, X.shape[0], q):
        Kb = kernel_block(X[s:s + q], C, kernel, sigma)
        U += Kb.T @ (Kb @ V)
    return U


def predict_multi(Xs, C, alpha, kernel: int, sigma: float, block_rows: int | None = None):
    """F = k(X*, C) alpha, alpha in R^{m x k} (Eq. (4))."""
    Xs = np.asarray(Xs, dtype=np.float64)
    q = _block_rows(C.shape[0], block_rows)
    out = np.empty((Xs.shape[0], alpha.shape[1]))
    for s in range(0, Xs.shape[0], q):
        out[s:s + q] = kernel_block(Xs[s:s + q], C, kernel, sigma) @ alpha
    return out


def fit_multi(X, Y, C, kernel: int, sigma: float, lam: float, iters: int,
              jitter: float = DEFAULT_JITTER):
    """Alg. 1 for the k columns of Y at once: one preconditioner (l.13-17),
    R = A^-T T^-T Knm^T Y (l.9), k CGs from 0 with per-column rho/gamma (l.10, reading c9;
    a column stops when its r^T r == 0), alpha = T^-1 A^-1 B (l.11)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    n, k = Y.shape
    T, A = preconditioner(C, kernel, sigma, lam, jitter)

    def su(U, B, trans):
        return sla.solve_triangular(U, B, lower=False, trans="T" if trans else "N")

    def linop(B):
        V = su(A, B, False)
        Cm = knm_t_knm_mat(X, C, su(T, V, False), kernel, sigma)
        return su(A, su(T, Cm, True) + lam * n * V, True)

    q = _block_rows(C.shape[0], None)
    KtY = np.zeros((C.shape[0], k))
    for s in range(0, n, q):
        KtY += kernel_block(X[s:s + q], C, kernel, sigma).T @ Y[s:s + q]
    R = su(A, su(T, KtY, True), True)
    Bx = np.zeros_like(R)
    Rr = R.copy()
    Pp = Rr.copy()
    rho = np.einsum("ij,ij->j", Rr, Rr)
    active = rho != 0.0
    for it in range(1, iters + 1):
        if not active.any():
            break
        Q = linop(Pp)
        gamma = np.einsum("ij,ij->j", Pp, Q)
        bad = active & (~(gamma > 0.0) | ~np.isfinite(gamma))
        if bad.any():
            raise NonFinite(it)
        a = np.where(active, rho / np.where(active, gamma, 1.0), 0.0)
        Bx = Bx + a * Pp
        Rr = Rr - a * Q
        rho_new = np.einsum("ij,ij->j", Rr, Rr)
        if not np.all(np.isfinite(rho_new[active])):
            raise NonFinite(it)
        beta = np.where(active, rho_new / np.where(active, rho, 1.0), 0.0)
        Pp = np.where(active, Rr + beta * Pp, Pp)
        rho = np.where(active, rho_new, rho)
        active = active & (rho_new != 0.0)
    return su(T, su(A, Bx, False), False)

