"""Falkon CPU oracle — plain, slow, fp64, written from the paper (arXiv 2006.10350).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.
The CUDA product path (``paper_2006_10350_b200``) never imports, links or executes
anything under ``oracle/``; the two share no code.

Every function follows one passage of PAPER.md (cited as ``PAPER.md:<line>``) and
the readings of SURVEY.md §8(c) / DESIGN.md ("Readings of the paper").  Inputs are
the fp32 arrays of ``synth`` upcast EXACTLY to fp64; all arithmetic is fp64.

Pins (tests/test_oracle.py, ``-m "not gpu"``):
  kernel_block      analytic values (tests/golden/kernel_values.txt), brute force
  knm_vec / knm_t_vec / knm_t_knm_vec
                    pure-Python brute force on tiny inputs, unit vectors, batching
                    invariance, self-adjointness, sigma->inf closed form
  preconditioner    T^T T = Kmm + delta I, A^T A = T T^T/m + lam I, whitening,
                    separated-centers closed form (T = I, A = sqrt(1/m+lam) I), m = 1
  conjugate_gradient  identity / 2I / random SPD vs direct solve
  linop             equals the dense Eq. (8) operator; C = X gives n*I exactly
  fit               C = X identity (one step = (Knn + n lam I)^-1 y);
                    n = m = 1 closed form; t >= m equals the Eq. (5) direct solve
  predict           alpha = 0, brute force
No function of this module is "parity unpinned"; the fit at the configured small t
has no closed form and is pinned only through the pieces above.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import scipy.linalg as sla

__all__ = ["GAUSSIAN", "LAPLACIAN", "DEFAULT_JITTER", "NotPositiveDefinite", "NonFinite",
           "sqdist", "kernel_block", "knm_vec", "knm_t_vec", "knm_t_knm_vec", "kmm",
           "preconditioner", "linop", "rhs", "conjugate_gradient", "fit", "predict"]

GAUSSIAN = 0
LAPLACIAN = 1

DEFAULT_JITTER = 1e-8        # SURVEY.md reading c6: delta added to diag(Kmm)
DIRECT_DIFF_MAX_D = 32       # oracle uses direct differences up to this d


class NotPositiveDefinite(RuntimeError):
    """Cholesky failure: which factor (0 = T, 1 = A)."""

    def __init__(self, factor: int):
        super().__init__(f"Cholesky failed on factor {'TA'[factor]}")
        self.factor = factor


class NonFinite(RuntimeError):
    """CG breakdown: p^T q <= 0 or non-finite at iteration `it` (SURVEY.md reading c9)."""

    def __init__(self, it: int):
        super().__init__(f"CG non-finite / non-positive curvature at iteration {it}")
        self.iteration = it


# --------------------------------------------------------------------------------------
# Kernel (PAPER.md:83 Gaussian; Laplacian = SURVEY.md reading c7)
# --------------------------------------------------------------------------------------
def sqdist(X1: np.ndarray, X2: np.ndarray, direct: bool | None = None) -> np.ndarray:
    """||x1_i - x2_j||^2 in fp64.  Direct differences for d <= 32 (or direct=True); for
    larger d the norm expansion ||x||^2 - 2 x.x' + ||x'||^2 clamped at 0
    (reading c8)."""
    X1 = np.asarray(X1, dtype=np.float64)
    X2 = np.asarray(X2, dtype=np.float64)
    d = X1.shape[1]
    if direct is None:
        direct = d <= DIRECT_DIFF_MAX_D
    if direct:
        # D_ij = sum_k (x1_ik - x2_jk)^2, k in order.  Column chunks of X2 with in-place
        # ufuncs keep the temporaries cache-sized (the same operations per element).
        n1, n2 = X1.shape[0], X2.shape[0]
        D = np.zeros((n1, n2), dtype=np.float64)
        X2T = np.ascontiguousarray(X2.T)
        cw = max(1, min(n2, (1 << 18) // max(n1, 1)))
        diff = np.empty((n1, cw), dtype=np.float64)
        for j0 in range(0, n2, cw):
            j1 = min(n2, j0 + cw)
            Dv, dv = D[:, j0:j1], diff[:, :j1 - j0]
            for k in range(d):
                np.subtract(X1[:, k:k + 1], X2T[k, None, j0:j1], out=dv)
                np.multiply(dv, dv, out=dv)
                Dv += dv
        return D
    n1 = np.einsum("ij,ij->i", X1, X1)
    n2 = np.einsum("ij,ij->i", X2, X2)
    D = n1[:, None] + n2[None, :] - 2.0 * (X1 @ X2.T)
    return np.maximum(D, 0.0)


def kernel_block(X1, X2, kernel: int, sigma: float) -> np.ndarray:
    """k(X1, X2): Gaussian exp(-||x-x'||^2 / (2 sigma^2));
    Laplacian exp(-||x-x'|| / sigma) (reading c7; always by direct differences, since
    the square root amplifies the expansion's cancellation residue)."""
    D = sqdist(X1, X2, direct=True if kernel == LAPLACIAN else None)
    if kernel == GAUSSIAN:
        return np.exp(-D / (2.0 * sigma * sigma))
    if kernel == LAPLACIAN:
        return np.exp(-np.sqrt(D) / sigma)
    raise ValueError(f"unknown kernel {kernel}")


# --------------------------------------------------------------------------------------
# Blockwise products, Knm never stored
# --------------------------------------------------------------------------------------
def _block_rows(m: int, block_rows: int | None) -> int:
    if block_rows is not None:
        return max(1, int(block_rows))
    return max(1, min(4096, (1 << 23) // max(m, 1)))


def knm_vec(X, C, v, kernel: int, sigma: float, block_rows: int | None = None) -> np.ndarray:
    """w = Knm v, row block by row block: w_b = k(X_b, C) v."""
    X = np.asarray(X, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    q = _block_rows(C.shape[0], block_rows)
    w = np.empty(X.shape[0], dtype=np.float64)
    for s in range(0, X.shape[0], q):
        w[s:s + q] = kernel_block(X[s:s + q], C, kernel, sigma) @ v
    return w


def knm_t_vec(X, C, w, kernel: int, sigma: float, block_rows: int | None = None,
              workers: int = 1) -> np.ndarray:
    """u = Knm^T w = sum_b k(X_b, C)^T w_b (Alg. 1 line 9, reading c2).
    ``workers > 1``: the row blocks are split over forked processes (as knm_t_knm_vec)."""
    X = np.asarray(X, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    q = _block_rows(C.shape[0], block_rows)
    if workers > 1 and X.shape[0] > q:
        return _pool_sum(X, C, w, kernel, sigma, q, workers, "t")
    return _kt_range((X, C, w, kernel, sigma, q, 0, X.shape[0]))


def _kt_range(args):
    X, C, w, kernel, sigma, q, lo, hi = args
    u = np.zeros(C.shape[0], dtype=np.float64)
    for s in range(lo, hi, q):
        e = min(s + q, hi)
        u += kernel_block(X[s:e], C, kernel, sigma).T @ w[s:e]
    return u


def _ktkv_range(args):
    X, C, v, kernel, sigma, q, lo, hi = args
    u = np.zeros(C.shape[0], dtype=np.float64)
    for s in range(lo, hi, q):
        Kb = kernel_block(X[s:min(s + q, hi)], C, kernel, sigma)
        u += Kb.T @ (Kb @ v)
    return u


_POOL_STATE = {}


def _pool_worker(bounds):
    st = _POOL_STATE
    fn = _kt_range if st["op"] == "t" else _ktkv_range
    return fn((st["X"], st["C"], st["v"], st["kernel"], st["sigma"], st["q"],
               bounds[0], bounds[1]))


def _pool_sum(X, C, v, kernel, sigma, q, workers, op):
    """Row blocks split over `workers` forked processes; each sums its own blocks
    (Knm^T(Knm v) for op "tkv", Knm^T v for op "t"); the per-worker sums are added in
    worker order."""
    n = X.shape[0]
    nblk = -(-n // q)
    per = -(-nblk // workers)
    bounds = [(i * per * q, min(n, (i + 1) * per * q)) for i in range(workers) if i * per * q < n]
    _POOL_STATE.update(X=X, C=C, v=v, kernel=kernel, sigma=sigma, q=q, op=op)
    import multiprocessing as mp
    try:
        with ProcessPoolExecutor(max_workers=len(bounds), mp_context=mp.get_context("fork"),
                                 initializer=_limit_blas_threads) as ex:
            parts = list(ex.map(_pool_worker, bounds))
    finally:
        _POOL_STATE.clear()
    u = np.zeros(C.shape[0], dtype=np.float64)
    for p in parts:
        u += p
    return u


def knm_t_knm_vec(X, C, v, kernel: int, sigma: float, block_rows: int | None = None,
                  workers: int = 1) -> np.ndarray:
    """u = Knm^T (Knm v) = sum_b k(X_b, C)^T (k(X_b, C) v).

    ``workers > 1`` splits the row blocks over forked processes (each sums its own
    blocks; the per-worker sums are added in worker order).  Used to time the oracle on
    all host cores (bench.py cpu_baseline) and for large parity runs; the arithmetic of
    every block is unchanged."""
    X = np.asarray(X, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    q = _block_rows(C.shape[0], block_rows)
    if workers <= 1 or X.shape[0] <= q:
        return _ktkv_range((X, C, v, kernel, sigma, q, 0, X.shape[0]))
    return _pool_sum(X, C, v, kernel, sigma, q, workers, "tkv")


def _limit_blas_threads():
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(1)
    except Exception:  # pragma: no cover - threadpoolctl is optional
        pass
    os.environ["OMP_NUM_THREADS"] = "1"


# --------------------------------------------------------------------------------------
# Preconditioner, Alg. 1 lines 13-17, Eq. (7)
# --------------------------------------------------------------------------------------
def kmm(C, kernel: int, sigma: float) -> np.ndarray:
    """K_mm = k(X_m, X_m) in fp64 (Alg. 1 line 14; fp64 as PAPER.md:480).
    Filled row block by row block into one m x m array (each block is kernel_block of
    those rows against all centres), so the peak memory is one m^2 buffer plus a block."""
    C = np.asarray(C, dtype=np.float64)
    m = C.shape[0]
    K = np.empty((m, m), dtype=np.float64)
    q = _block_rows(m, None)
    for s in range(0, m, q):
        K[s:s + q] = kernel_block(C[s:s + q], C, kernel, sigma)
    return K


# Block size of the blocked Cholesky / triangular solves below.  LAPACK and BLAS calls on
# whole m x m matrices go through scipy's LP64 (32-bit index) OpenBLAS, whose index
# arithmetic overflows once m^2 > 2^31 (m > 46,340: dpotrf / dtrsv segfault at m = 5e4);
# every LAPACK call here is on a NB x NB diagonal block, and the large products are numpy
# matmuls (ILP64 OpenBLAS) on views of at most NB rows or columns.
CHOL_NB = 2048


def _chol_upper_inplace(M: np.ndarray, nb: int = CHOL_NB) -> np.ndarray:
    """Upper R with R^T R = M, computed IN the C-contiguous buffer of M (its upper triangle
    is read; the strict lower triangle is zeroed).  Textbook right-looking blocked Cholesky
    (the blocked POTRF of App. C Alg. 4, in core): for each diagonal
    block k
        R_kk = chol(M_kk)                         (LAPACK dpotrf on an nb x nb block)
        R_k,j = R_kk^-T M_k,j        (j > k)      (triangular solve, the panel row)
        M_i,j -= R_k,i^T R_k,j       (k < i <= j) (trailing update, upper blocks only)
    Raises np.linalg.LinAlgError on a non-positive pivot, as LAPACK."""
    assert M.flags["C_CONTIGUOUS"] and M.shape[0] == M.shape[1]
    m = M.shape[0]
    for k0 in range(0, m, nb):
        k1 = min(m, k0 + nb)
        Rkk = sla.cholesky(M[k0:k1, k0:k1], lower=False, check_finite=False)
        M[k0:k1, k0:k1] = Rkk
        if k1 == m:
            break
        M[k0:k1, k1:] = sla.solve_triangular(Rkk, M[k0:k1, k1:], trans="T", lower=False,
                                             check_finite=False)
        P = M[k0:k1, :]  # panel row: R_k,* for columns >= k1
        for j0 in range(k1, m, nb):
            j1 = min(m, j0 + nb)
            M[k1:j1, j0:j1] -= P[:, k1:j1].T @ P[:, j0:j1]
    for i0 in range(0, m, nb):  # zero the strict lower triangle
        i1 = min(m, i0 + nb)
        M[i0:i1, :i0] = 0.0
        blk = M[i0:i1, i0:i1]
        blk[np.tril_indices(i1 - i0, -1)] = 0.0
    return M


def preconditioner(C, kernel: int, sigma: float, lam: float, jitter: float = DEFAULT_JITTER):
    """(T, A), both UPPER triangular with
        T^T T = K_mm + delta I                       (line 15; K_mm = T^T T)
        A^T A = (1/m) T T^T + lam I                  (lines 16-17; reading c3/c4)
    delta = `jitter` (reading c6).  Memory-lean but the same arithmetic as the formulas:
    delta and lam are added to the diagonals in place (adding the zero off-diagonal
    entries of delta I / lam I is exact), each Cholesky overwrites its input buffer, so
    the peak is two m x m fp64 buffers (T and A)."""
    K = kmm(C, kernel, sigma)
    m = K.shape[0]
    diag = np.arange(m)
    K[diag, diag] += jitter
    try:
        T = _chol_upper_inplace(K)
    except np.linalg.LinAlgError:
        raise NotPositiveDefinite(0) from None
    del K
    M = _upper_times_transpose(T)
    M /= m
    M[diag, diag] += lam
    try:
        A = _chol_upper_inplace(M)
    except np.linalg.LinAlgError:
        raise NotPositiveDefinite(1) from None
    return T, A


def _upper_times_transpose(T: np.ndarray, nb: int = CHOL_NB) -> np.ndarray:
    """T T^T for upper-triangular T, by nb x nb blocks (numpy's whole-matrix T @ T.T
    segfaults in its BLAS for m > 46,340, see CHOL_NB): block (I, J), J <= I, is
    T[I, i0:] @ T[J, i0:]^T (the columns k < i0 of T[I, :] are exact zeros), mirrored."""
    m = T.shape[0]
    M = np.empty((m, m), dtype=np.float64)
    for i0 in range(0, m, nb):
        i1 = min(m, i0 + nb)
        for j0 in range(0, i1, nb):
            j1 = min(m, j0 + nb)
            blk = T[i0:i1, i0:] @ T[j0:j1, i0:].T
            M[i0:i1, j0:j1] = blk
            M[j0:j1, i0:i1] = blk.T
    return M


def _solve_upper(U, b, trans: bool, nb: int = CHOL_NB):
    """U x = b (trans=False) or U^T x = b (trans=True), U upper triangular: block back
    (forward) substitution, LAPACK dtrsv on nb x nb diagonal blocks and numpy mat-vecs
    for the off-diagonal blocks (see CHOL_NB)."""
    m = U.shape[0]
    x = np.array(b, dtype=np.float64, copy=True)
    starts = list(range(0, m, nb))
    if not trans:  # U x = b: last block first
        for i0 in reversed(starts):
            i1 = min(m, i0 + nb)
            if i1 < m:
                x[i0:i1] -= U[i0:i1, i1:] @ x[i1:]
            x[i0:i1] = sla.solve_triangular(U[i0:i1, i0:i1], x[i0:i1], lower=False,
                                            check_finite=False)
    else:  # U^T x = b: first block first
        for i0 in starts:
            i1 = min(m, i0 + nb)
            if i0 > 0:
                x[i0:i1] -= U[:i0, i0:i1].T @ x[:i0]
            x[i0:i1] = sla.solve_triangular(U[i0:i1, i0:i1], x[i0:i1], lower=False,
                                            trans="T", check_finite=False)
    return x


# --------------------------------------------------------------------------------------
# Alg. 1, LinOp read as Eq. (9) (reading c1)
# --------------------------------------------------------------------------------------
def linop(beta, X, C, T, A, lam: float, kernel: int, sigma: float, n_global: int | None = None,
          block_rows: int | None = None, workers: int = 1):
    """Alg. 1 lines 4-8 as Eq. (9):
        v = A^-1 beta                     (line 5)
        c = Knm^T Knm T^-1 v              (line 6)
        return A^-T (T^-T c + lam n v)    (line 7, Eq. (9) parenthesisation)"""
    n = X.shape[0] if n_global is None else n_global
    v = _solve_upper(A, beta, trans=False)
    c = knm_t_knm_vec(X, C, _solve_upper(T, v, trans=False), kernel, sigma, block_rows, workers)
    return _solve_upper(A, _solve_upper(T, c, trans=True) + lam * n * v, trans=True)


def rhs(X, y, C, T, A, kernel: int, sigma: float, block_rows: int | None = None,
        workers: int = 1):
    """R = A^-T T^-T Knm^T y  (Alg. 1 line 9, reading c2)."""
    c = knm_t_vec(X, C, y, kernel, sigma, block_rows, workers)
    return _solve_upper(A, _solve_upper(T, c, trans=True), trans=True)


def conjugate_gradient(op, b, t: int):
    """Textbook Hestenes-Stiefel CG from x0 = 0, exactly t iterations (Alg. 1 line 10,
    PAPER.md:115; reading c9: stop early only if r^T r == 0 exactly; error if p^T A p <= 0
    or non-finite).  Returns (x, iterations_run)."""
    x = np.zeros_like(b, dtype=np.float64)
    r = np.array(b, dtype=np.float64, copy=True)
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


def fit(X, y, C, kernel: int, sigma: float, lam: float, iters: int,
        jitter: float = DEFAULT_JITTER, block_rows: int | None = None, return_info: bool = False,
        workers: int = 1):
    """Falkon, Alg. 1: preconditioner, R, CG(LinOp, R, t),
    alpha = T^-1 A^-1 beta.  C (= X_m) is an input (sampling lives in synth, reading c11).
    `workers` only parallelises the row blocks of the products (RHS and LinOp)."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    T, A = preconditioner(C, kernel, sigma, lam, jitter)
    R = rhs(X, y, C, T, A, kernel, sigma, block_rows, workers)
    beta, it = conjugate_gradient(
        lambda b: linop(b, X, C, T, A, lam, kernel, sigma, block_rows=block_rows, workers=workers),
        R, iters)
    alpha = _solve_upper(T, _solve_upper(A, beta, trans=False), trans=False)
    if return_info:
        return alpha, {"T": T, "A": A, "R": R, "beta": beta, "iters_run": it}
    return alpha


def predict(Xs, C, alpha, kernel: int, sigma: float, block_rows: int | None = None):
    """f(x) = sum_j alpha_j k(x, c_j)  (Eq. (4))."""
    return knm_vec(Xs, C, alpha, kernel, sigma, block_rows)
