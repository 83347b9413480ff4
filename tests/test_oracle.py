"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it pins.  None of them re-types the oracle's formula:
they use closed forms, brute force in pure Python, invariants, or a DIFFERENT
construction (e.g. the dense Eq. (5) / Eq. (8) systems) of the same quantity.
"""
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
G, L = oracle.GAUSSIAN, oracle.LAPLACIAN


def _rng(seed=0):
    return np.random.default_rng(seed)


# ------------------------------------------------------------------ kernel values
def _golden_kernel_rows():
    rows = []
    with open(os.path.join(GOLD, "kernel_values.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            kname, sig, x, xp, exp_val = line.split()[:5]
            rows.append((kname, float(sig), [float(t) for t in x.split(",")],
                         [float(t) for t in xp.split(",")], float(exp_val)))
    return rows


@pytest.mark.parametrize("row", _golden_kernel_rows())
def test_kernel_golden_values(row):
    """tests/golden/kernel_values.txt (reading c7)."""
    kname, sig, x, xp, expected = row
    k = oracle.kernel_block(np.array([x]), np.array([xp]), G if kname == "gaussian" else L, sig)
    assert abs(k[0, 0] - expected) <= 4e-16 * max(1.0, expected)


def _brute_K(X, C, kernel, sigma):
    K = []
    for x in X.tolist():
        row = []
        for c in C.tolist():
            d2 = sum((a - b) ** 2 for a, b in zip(x, c))
            row.append(math.exp(-d2 / (2 * sigma * sigma)) if kernel == G
                       else math.exp(-math.sqrt(d2) / sigma))
        K.append(row)
    return K


@pytest.mark.parametrize("kernel", [G, L])
@pytest.mark.parametrize("d", [1, 5, 8, 40])
def test_kernel_block_brute_force(kernel, d):
    """Both sqdist branches (direct differences d<=32, norm expansion d>32)
    against a pure-Python loop; symmetry and unit diagonal of k(X,X)."""
    rng = _rng(d)
    X = rng.standard_normal((13, d)).astype(np.float32)
    C = rng.standard_normal((7, d)).astype(np.float32)
    sigma = 1.3 if d < 40 else 6.0
    K = oracle.kernel_block(X, C, kernel, sigma)
    Kb = np.array(_brute_K(X.astype(np.float64), C.astype(np.float64), kernel, sigma))
    tol = 1e-14 if d <= 32 else 5e-12
    assert np.max(np.abs(K - Kb)) <= tol
    Kxx = oracle.kernel_block(X, X, kernel, sigma)
    assert np.array_equal(Kxx, Kxx.T) or np.max(np.abs(Kxx - Kxx.T)) < 1e-15
    assert np.allclose(np.diag(Kxx), 1.0, rtol=0, atol=1e-12)


# ------------------------------------------------------------------ products
def _brute_products(X, C, v, kernel, sigma):
    K = _brute_K(X, C, kernel, sigma)
    w = [sum(Kij * vj for Kij, vj in zip(row, v)) for row in K]
    u = [sum(K[i][j] * w[i] for i in range(len(K))) for j in range(len(C))]
    return np.array(w), np.array(u)


@pytest.mark.parametrize("kernel", [G, L])
def test_products_brute_force(kernel):
    """Knm v, Knm^T w, Knm^T(Knm v) against a pure-Python triple loop (n<=64, m<=16, d<=8)."""
    rng = _rng(1)
    X = rng.standard_normal((64, 8)).astype(np.float32).astype(np.float64)
    C = X[rng.choice(64, 16, replace=False)]
    v = rng.standard_normal(16)
    w_b, u_b = _brute_products(X, C, v.tolist(), kernel, 1.7)
    w = oracle.knm_vec(X, C, v, kernel, 1.7, block_rows=5)
    u = oracle.knm_t_knm_vec(X, C, v, kernel, 1.7, block_rows=5)
    u2 = oracle.knm_t_vec(X, C, w_b, kernel, 1.7, block_rows=9)
    assert np.max(np.abs(w - w_b)) <= 1e-13 * np.max(np.abs(w_b))
    assert np.max(np.abs(u - u_b)) <= 1e-13 * np.max(np.abs(u_b))
    assert np.max(np.abs(u2 - u_b)) <= 1e-13 * np.max(np.abs(u_b))


def test_products_special_vectors():
    """v = 0 -> 0; w = e_i -> kernel row i; v = e_j -> column."""
    rng = _rng(2)
    X = rng.standard_normal((50, 4))
    C = X[:10]
    assert np.all(oracle.knm_t_knm_vec(X, C, np.zeros(10), G, 1.0) == 0.0)
    e = np.zeros(50)
    e[7] = 1.0
    row = oracle.knm_t_vec(X, C, e, G, 1.0)
    brute = np.array(_brute_K(X[7:8], C, G, 1.0)[0])
    assert np.max(np.abs(row - brute)) < 1e-15
    ej = np.zeros(10)
    ej[3] = 1.0
    col = oracle.knm_vec(X, C, ej, G, 1.0)
    brute_col = np.array([r[3] for r in _brute_K(X, C, G, 1.0)])
    assert np.max(np.abs(col - brute_col)) < 1e-15


def test_products_batching_and_workers_invariance():
    """Result independent of the row-batch size q and of the worker split."""
    rng = _rng(3)
    X = rng.standard_normal((300, 6))
    C = X[rng.choice(300, 40, replace=False)]
    v = rng.standard_normal(40)
    ref = oracle.knm_t_knm_vec(X, C, v, G, 1.2, block_rows=300)
    for q in (7, 64):
        u = oracle.knm_t_knm_vec(X, C, v, G, 1.2, block_rows=q)
        assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))
    u = oracle.knm_t_knm_vec(X, C, v, G, 1.2, block_rows=16, workers=3)
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_products_self_adjoint_and_psd():
    """<KtKv(v1), v2> = <v1, KtKv(v2)> and v^T KtKv(v) = ||Knm v||^2 >= 0."""
    rng = _rng(4)
    X = rng.standard_normal((200, 9))
    C = X[:30]
    v1, v2 = rng.standard_normal(30), rng.standard_normal(30)
    a = oracle.knm_t_knm_vec(X, C, v1, G, 1.0) @ v2
    b = v1 @ oracle.knm_t_knm_vec(X, C, v2, G, 1.0)
    assert abs(a - b) <= 1e-12 * abs(a)
    w = oracle.knm_vec(X, C, v1, G, 1.0)
    assert abs(v1 @ oracle.knm_t_knm_vec(X, C, v1, G, 1.0) - w @ w) <= 1e-12 * (w @ w)


def test_products_sigma_infinity_closed_form():
    """sigma -> inf: K -> 1 (all ones), so Knm^T Knm v = n (sum v) 1 (SURVEY.md §8(c) pins)."""
    rng = _rng(5)
    X = rng.standard_normal((500, 9))
    C = X[:25]
    v = rng.random(25)
    u = oracle.knm_t_knm_vec(X, C, v, G, 1e7)
    assert np.max(np.abs(u - 500 * v.sum())) <= 1e-9 * 500 * v.sum()


# ------------------------------------------------------------------ preconditioner
def test_preconditioner_factor_identities():
    """T^T T = Kmm + delta I, A^T A = T T^T/m + lam I (Eq. (7)); whitening
    T^-T Kmm T^-1 ~ I; Kmm symmetric PSD (north_star)."""
    cfg, X, y, C = synth.make_problem("tiny")
    C = C.astype(np.float64)
    m = C.shape[0]
    K = oracle.kmm(C, G, 1.0)
    assert np.array_equal(K, K.T)
    assert np.linalg.eigvalsh(K).min() >= -1e-14 * m
    T, A = oracle.preconditioner(C, G, 1.0, 1e-6, jitter=1e-8)
    assert np.allclose(np.tril(T, -1), 0) and np.allclose(np.tril(A, -1), 0)
    assert np.max(np.abs(T.T @ T - (K + 1e-8 * np.eye(m)))) <= 1e-13
    M = T @ T.T / m + 1e-6 * np.eye(m)
    assert np.max(np.abs(A.T @ A - M)) <= 1e-14
    Ti = np.linalg.inv(T)
    W = Ti.T @ K @ Ti
    assert np.max(np.abs(W - np.eye(m))) <= 1e-6


def test_preconditioner_separated_centers_closed_form():
    """Centers far apart relative to sigma -> Kmm = I exactly -> T = sqrt(1+delta) I and
    A = sqrt((1+delta)/m + lam) I (SPEC S:211 analogue for the Gaussian kernel)."""
    m, lam, delta = 6, 1e-3, 1e-8
    C = 10.0 * np.eye(m)
    T, A = oracle.preconditioner(C, G, 0.1, lam, jitter=delta)
    assert np.allclose(T, math.sqrt(1 + delta) * np.eye(m), rtol=0, atol=1e-15)
    assert np.allclose(A, math.sqrt((1 + delta) / m + lam) * np.eye(m), rtol=0, atol=1e-15)


def test_preconditioner_m1():
    """m = 1: T = 1, A = sqrt(1 + lam), delta = 0."""
    T, A = oracle.preconditioner(np.array([[0.3, -2.0]]), L, 1.0, 0.25, jitter=0.0)
    assert T[0, 0] == 1.0 and abs(A[0, 0] - math.sqrt(1.25)) < 1e-16


def test_preconditioner_not_pd_raises():
    """Duplicate centers + delta = 0 + lam = 0 -> singular Kmm -> NotPositiveDefinite(T)
    (SURVEY.md §8(b) ENOTPD)."""
    C = np.array([[0.0, 1.0], [0.0, 1.0], [2.0, 2.0]])
    with pytest.raises(oracle.NotPositiveDefinite) as e:
        oracle.preconditioner(C, G, 1.0, 0.0, jitter=0.0)
    assert e.value.factor == 0


# ------------------------------------------------------------------ CG (Alg. 1 line 10)
def test_cg_identity_and_scaled():
    """op = I -> rhs after 1 step; op = 2I -> rhs/2."""
    b = _rng(6).standard_normal(12)
    x, it = oracle.conjugate_gradient(lambda p: p, b, 5)
    assert np.allclose(x, b, rtol=0, atol=1e-15) and it == 1
    x, it = oracle.conjugate_gradient(lambda p: 2 * p, b, 5)
    assert np.allclose(x, b / 2, rtol=0, atol=1e-15) and it == 1


def test_cg_random_spd():
    """Random SPD 20x20, t=20 vs direct solve, <= 1e-8."""
    rng = _rng(7)
    B = rng.standard_normal((20, 20))
    S = B @ B.T + 20 * np.eye(20)
    b = rng.standard_normal(20)
    x, _ = oracle.conjugate_gradient(lambda p: S @ p, b, 20)
    xs = np.linalg.solve(S, b)
    assert np.linalg.norm(x - xs) <= 1e-8 * np.linalg.norm(xs)


def test_cg_breakdown_raises():
    """Indefinite operator -> p^T A p <= 0 -> NonFinite(1) (reading c9)."""
    with pytest.raises(oracle.NonFinite):
        oracle.conjugate_gradient(lambda p: -p, np.ones(3), 3)


# ------------------------------------------------------------------ LinOp (Eq. (8)-(9))
def test_linop_equals_dense_eq8_operator():
    """LinOp(beta) = P^T (Knm^T Knm + lam n (Kmm + delta I)) P beta with P = T^-1 A^-1
    (Eq. (8); 1/sqrt(n) dropped, reading c5), built densely."""
    rng = _rng(8)
    n, m, d, sigma, lam, delta = 200, 30, 5, 1.0, 1e-3, 1e-8
    X = rng.standard_normal((n, d))
    C = X[rng.choice(n, m, replace=False)]
    T, A = oracle.preconditioner(C, G, sigma, lam, jitter=delta)
    Knm = np.array(_brute_K(X, C, G, sigma))
    Kmm = np.array(_brute_K(C, C, G, sigma)) + delta * np.eye(m)
    P = np.linalg.inv(T) @ np.linalg.inv(A)
    H = Knm.T @ Knm + lam * n * Kmm
    dense = P.T @ H @ P
    assert np.max(np.abs(dense - dense.T)) <= 1e-8 * np.max(np.abs(dense))
    for _ in range(3):
        beta = rng.standard_normal(m)
        got = oracle.linop(beta, X, C, T, A, lam, G, sigma)
        ref = dense @ beta
        assert np.linalg.norm(got - ref) <= 1e-8 * np.linalg.norm(ref)


def test_linop_literal_reading_breaks_identity():
    """Documents reading c1: the literal Alg. 1 line 7 A^-T T^-T c + lam n v is NOT the
    Eq. (9) operator (with C = X the Eq. (9) operator is exactly n I; the literal one is not)."""
    rng = _rng(9)
    n, d, sigma, lam = 60, 4, 1.0, 1e-3
    X = rng.standard_normal((n, d))
    T, A = oracle.preconditioner(X, G, sigma, lam, jitter=0.0)
    beta = rng.standard_normal(n)
    op = oracle.linop(beta, X, X, T, A, lam, G, sigma)
    assert np.linalg.norm(op - n * beta) <= 1e-9 * n * np.linalg.norm(beta)
    import scipy.linalg as sla
    v = sla.solve_triangular(A, beta, lower=False)
    c = oracle.knm_t_knm_vec(X, X, sla.solve_triangular(T, v, lower=False), G, sigma)
    literal = sla.solve_triangular(A, sla.solve_triangular(T, c, trans="T"), trans="T") + lam * n * v
    assert np.linalg.norm(literal - n * beta) > 1e-3 * n * np.linalg.norm(beta)


# ------------------------------------------------------------------ fit (Alg. 1) and predict (Eq. 4)
@pytest.mark.parametrize("kernel", [G, L])
def test_fit_C_equals_X_identity(kernel):
    """north_star identity: with m = n and C = X the preconditioned operator is n I, so one
    CG step gives alpha = (Knn + n lam I)^-1 y (KRR system)."""
    rng = _rng(10)
    n, d, sigma, lam = 150, 6, 1.5, 1e-3
    X = rng.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    y = np.sin(X[:, 0]) + 0.1 * rng.standard_normal(n)
    Knn = np.array(_brute_K(X, X, kernel, sigma))
    alpha_krr = np.linalg.solve(Knn + n * lam * np.eye(n), y)
    for t in (1, 3):
        alpha = oracle.fit(X, y, X, kernel, sigma, lam, t, jitter=0.0)
        assert np.linalg.norm(alpha - alpha_krr) <= 1e-9 * np.linalg.norm(alpha_krr)


def test_fit_scalar_closed_form():
    """n = m = 1: alpha = y / (1 + lam), delta = 0."""
    for lam in (0.0, 0.5, 3.0):
        a = oracle.fit(np.array([[0.2, 0.1]]), np.array([2.5]), np.array([[0.2, 0.1]]), G, 1.0,
                       lam, 4, jitter=0.0)
        assert abs(a[0] - 2.5 / (1 + lam)) <= 1e-15 * 2.5


def test_fit_many_iterations_equals_eq5_direct_solve():
    """t >> m: alpha solves (Knm^T Knm + lam n (Kmm + delta I)) alpha = Knm^T y (Eq. (5),
    PAPER.md:150-152)."""
    rng = _rng(11)
    n, m, d, sigma, lam, delta = 500, 30, 5, 1.0, 1e-4, 1e-8
    X = rng.standard_normal((n, d))
    C = X[rng.choice(n, m, replace=False)]
    y = np.sin(X.sum(1)) + 0.2 * rng.standard_normal(n)
    Knm = np.array(_brute_K(X, C, G, sigma))
    Kmm = np.array(_brute_K(C, C, G, sigma)) + delta * np.eye(m)
    alpha_direct = np.linalg.solve(Knm.T @ Knm + lam * n * Kmm, Knm.T @ y)
    alpha = oracle.fit(X, y, C, G, sigma, lam, 3 * m, jitter=delta)
    assert np.linalg.norm(alpha - alpha_direct) <= 1e-8 * np.linalg.norm(alpha_direct)


def test_fit_tiny_config_converges_toward_eq5():
    """The tiny config (BASELINE.json configs[0]) at t = 10 is close to, but not at, the
    Eq. (5) solution (1.5e-3): the oracle must run exactly t steps."""
    cfg, X, y, C = synth.make_problem("tiny")
    X, y, C = (a.astype(np.float64) for a in (X, y, C))
    a10 = oracle.fit(X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    a60 = oracle.fit(X, y, C, G, cfg.sigma, cfg.lam, 60)
    Knm = oracle.kernel_block(X, C, G, cfg.sigma)
    Kmm = oracle.kmm(C, G, cfg.sigma) + oracle.DEFAULT_JITTER * np.eye(cfg.m)
    direct = np.linalg.solve(Knm.T @ Knm + cfg.lam * cfg.n * Kmm, Knm.T @ y)
    e10 = np.linalg.norm(a10 - direct) / np.linalg.norm(direct)
    e60 = np.linalg.norm(a60 - direct) / np.linalg.norm(direct)
    assert 1e-5 < e10 < 5e-2
    assert e60 < 1e-7


def test_predict():
    """alpha = 0 -> 0; brute force k(X*, C) alpha (Eq. (4))."""
    rng = _rng(12)
    Xs = rng.standard_normal((20, 3))
    C = rng.standard_normal((7, 3))
    a = rng.standard_normal(7)
    assert np.all(oracle.predict(Xs, C, np.zeros(7), G, 1.0) == 0)
    brute = np.array([sum(k * aj for k, aj in zip(row, a)) for row in _brute_K(Xs, C, G, 0.8)])
    assert np.max(np.abs(oracle.predict(Xs, C, a, G, 0.8) - brute)) <= 1e-14


# ------------------------------------------------------------------ synthetic inputs
def test_synth_configs_match_table3():
    """synth.CONFIGS hyper-parameters = Table 3 (tests/golden/table3_hparams.txt)."""
    with open(os.path.join(GOLD, "table3_hparams.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, sig, lam, ep, d = line.split()
            c = synth.CONFIGS[name]
            assert c.sigma == float(sig) and c.lam == float(lam) and c.d == int(d)
            if name != "msd":
                assert c.iters == int(ep)
    assert synth.CONFIGS["msd"].iters == 20


def test_synth_random_access_and_distribution():
    """Any row range regenerates bit-identically; X ~ N(0,1); C subset of X."""
    X = synth.gen_X(5, 0, 1000, 7)
    assert np.array_equal(X[300:400], synth.gen_X(5, 300, 100, 7))
    assert abs(float(X.mean())) < 0.05 and abs(float(X.std()) - 1) < 0.05
    cfg, Xt, yt, Ct = synth.make_problem("tiny")
    idx = synth.center_indices(cfg.seed, cfg.n, cfg.m)
    assert len(np.unique(idx)) == cfg.m
    assert np.array_equal(Ct, Xt[idx])
    lo, hi = synth.shard_range(10, 3, 0), synth.shard_range(10, 3, 2)
    assert lo == (0, 4) and hi == (7, 10)


def test_synth_device_generator_matches_host():
    """synth.gen_X_torch (used for inputs too large for the host, e.g. TAXI) reproduces
    synth.gen_X bit for bit on the CPU torch backend."""
    torch = pytest.importorskip("torch")
    a = synth.gen_X(4, 987654321, 3000, 9)
    b = synth.gen_X_torch(4, 987654321, 3000, 9, device="cpu").numpy()
    assert np.array_equal(a, b)


def test_device_target_generator_matches_host():
    """synth.gen_y_torch (targets of device-generated X) reproduces synth.gen_y."""
    import torch
    X = synth.gen_X(4, 123456789, 5000, 9)
    for task in ("reg", "cls"):
        a = synth.gen_y(4, X, 123456789, task)
        b = synth.gen_y_torch(4, torch.from_numpy(X), 123456789, task, chunk_rows=1500).numpy()
        assert np.max(np.abs(a.astype(np.float64) - b)) <= 1e-6


def test_blocked_cholesky_and_solves_match_lapack():
    """The oracle's blocked Cholesky / triangular solves (used so that no LAPACK call sees an
    m x m matrix: scipy's LP64 OpenBLAS overflows past m = 46,340) equal unblocked LAPACK on
    SPD matrices, for block sizes that leave ragged last blocks."""
    import scipy.linalg as sla
    from oracle import falkon_oracle as fo
    rng = np.random.default_rng(11)
    for m, nb in [(301, 7), (130, 64), (64, 64), (9, 2)]:
        B = rng.standard_normal((m, m))
        M = B @ B.T + m * np.eye(m)
        R0 = sla.cholesky(M, lower=False)
        R = fo._chol_upper_inplace(M.copy(), nb)
        assert np.allclose(R, R0, rtol=0, atol=1e-12 * np.abs(R0).max())
        assert np.all(np.tril(R, -1) == 0.0)
        b = rng.standard_normal(m)
        for trans in (False, True):
            x = fo._solve_upper(R0, b, trans, nb)
            x0 = sla.solve_triangular(R0, b, lower=False, trans="T" if trans else "N")
            assert np.allclose(x, x0, rtol=1e-12, atol=1e-12)
    with pytest.raises(np.linalg.LinAlgError):
        fo._chol_upper_inplace(-np.eye(5), 2)


def test_blocked_upper_times_transpose():
    """T T^T by blocks (the oracle's LAUUM, avoiding numpy's whole-matrix product that crashes
    past m = 46,340) equals the plain product and is exactly symmetric."""
    from oracle import falkon_oracle as fo
    rng = np.random.default_rng(12)
    for m, nb in [(301, 7), (129, 64), (40, 2048)]:
        T = np.triu(rng.standard_normal((m, m)))
        M = fo._upper_times_transpose(T, nb)
        assert np.allclose(M, T @ T.T, rtol=0, atol=1e-12 * m)
        assert np.array_equal(M, M.T)
