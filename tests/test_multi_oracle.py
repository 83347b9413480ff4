"""Pins of the multi-output oracle (oracle/multi_oracle.py), -m "not gpu":
the matrix-form code against the single-output oracle (a different code path) column by
column, k = 1, and column permutation."""
import numpy as np
import pytest

import oracle
import synth
from oracle import multi

G, L = oracle.GAUSSIAN, oracle.LAPLACIAN


def _problem(n=400, m=40, d=5, k=4, seed=0):
    X = synth.gen_X(seed, 0, n, d)
    idx = synth.center_indices(seed, n, m)
    r = np.random.default_rng(seed)
    Y = (np.sin(X[:, :1] + np.arange(k)[None, :]) + 0.1 * r.standard_normal((n, k))).astype(np.float32)
    return X, Y, X[idx].copy()


@pytest.mark.parametrize("kernel", [G, L])
def test_product_columns_equal_single(kernel):
    X, _, C = _problem()
    V = np.random.default_rng(1).standard_normal((C.shape[0], 6))
    U = multi.knm_t_knm_mat(X, C, V, kernel, 1.3, block_rows=57)
    for c in range(V.shape[1]):
        u = oracle.knm_t_knm_vec(X, C, V[:, c], kernel, 1.3)
        assert np.linalg.norm(U[:, c] - u) <= 1e-13 * np.linalg.norm(u)


def test_fit_columns_equal_single_fit():
    """Alg. 1 per column (multi-class as k outputs)."""
    X, Y, C = _problem()
    lam, t = 1e-4, 7
    A = multi.fit_multi(X, Y, C, G, 1.3, lam, t)
    for c in range(Y.shape[1]):
        a = oracle.fit(X, Y[:, c], C, G, 1.3, lam, t)
        assert np.linalg.norm(A[:, c] - a) <= 1e-10 * np.linalg.norm(a)
    Xs = synth.gen_X(5, 0, 50, 5)
    F = multi.predict_multi(Xs, C, A, G, 1.3)
    assert np.allclose(F[:, 2], oracle.predict(Xs, C, A[:, 2], G, 1.3), rtol=1e-12, atol=1e-12)


def test_k1_and_permutation_and_zero_column():
    X, Y, C = _problem(k=3)
    A1 = multi.fit_multi(X, Y[:, :1], C, G, 1.3, 1e-4, 5)
    assert np.allclose(A1[:, 0], oracle.fit(X, Y[:, 0], C, G, 1.3, 1e-4, 5), rtol=1e-10, atol=1e-12)
    perm = [2, 0, 1]
    A = multi.fit_multi(X, Y, C, G, 1.3, 1e-4, 5)
    Ap = multi.fit_multi(X, Y[:, perm], C, G, 1.3, 1e-4, 5)
    assert np.allclose(Ap, A[:, perm], rtol=1e-12, atol=1e-13)
    Y0 = Y.copy()
    Y0[:, 1] = 0.0  # a zero column stops at once (r^T r == 0, reading c9) and gives alpha = 0
    A0 = multi.fit_multi(X, Y0, C, G, 1.3, 1e-4, 5)
    assert np.all(A0[:, 1] == 0.0) and np.allclose(A0[:, 0], A[:, 0], rtol=1e-12, atol=1e-13)
