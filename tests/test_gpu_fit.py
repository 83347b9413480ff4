"""GPU parity of the fp64 preconditioner (a9), the triangular solves (a7), the full Falkon fit
(Alg. 1) and predict (Eq. (4)) against the oracle.

Bars (north_star): fitted alpha and predictions within 1e-3 relative error of the oracle.
The preconditioner factors are compared at fp64 level (they are pure fp64 on both sides).
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = pytest.mark.gpu
G, L = oracle.GAUSSIAN, oracle.LAPLACIAN


def _build(ctx, C, kernel, sigma, lam, jitter):
    import torch
    m = C.shape[0]
    P = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    dT, dA = zeros(m), zeros(m)
    W = zeros(ctx.precond_work_elems(m))
    info = ctx.precond_build(dev(C), kernel, sigma, lam, jitter, P, dT, dA, W)
    Ph, dTh, dAh = host(P), host(dT), host(dA)
    T = np.triu(Ph, 1) + np.diag(dTh)
    A = (np.tril(Ph, -1) + np.diag(dAh)).T
    return T, A, (P, dT, dA, W), info


@pytest.mark.parametrize("m,d,kernel,sigma", [(100, 8, G, 1.0), (300, 9, G, 1.0),
                                               (257, 28, L, 3.8), (129, 90, G, 7.0),
                                               (1, 3, G, 1.0), (600, 5, G, 1.5)])
def test_preconditioner_parity(ctx, m, d, kernel, sigma):
    lam, jit = 1e-6, 1e-8
    C = synth.gen_X(m + d, 0, m, d)
    T, A, _, info = _build(ctx, C, kernel, sigma, lam, jit)
    To, Ao = oracle.preconditioner(C, kernel, sigma, lam, jit)
    assert info["failed_factor"] == -1
    assert np.max(np.abs(T - To)) <= 1e-9 * max(1.0, np.max(np.abs(To)))
    assert np.max(np.abs(A - Ao)) <= 1e-8 * max(1.0, np.max(np.abs(Ao)))
    K = oracle.kmm(C, kernel, sigma) + jit * np.eye(m)
    assert np.max(np.abs(T.T @ T - K)) <= 1e-11
    M = T @ T.T / m + lam * np.eye(m)
    assert np.max(np.abs(A.T @ A - M)) <= 1e-11


def test_preconditioner_separated_centers_closed_form(ctx):
    m, lam, delta = 8, 1e-3, 1e-8
    C = (10.0 * np.eye(m)).astype(np.float32)
    T, A, _, _ = _build(ctx, C, G, 0.1, lam, delta)
    assert np.allclose(T, math.sqrt(1 + delta) * np.eye(m), rtol=0, atol=1e-15)
    assert np.allclose(A, math.sqrt((1 + delta) / m + lam) * np.eye(m), rtol=0, atol=1e-15)


def test_preconditioner_not_pd(ctx):
    from paper_2006_10350_b200 import FalkonError
    C = np.array([[0.0, 1.0], [0.0, 1.0], [2.0, 2.0]], dtype=np.float32)
    with pytest.raises(FalkonError) as e:
        _build(ctx, C, G, 1.0, 0.0, 0.0)
    assert e.value.code == 2 and e.value.info["failed_factor"] == 0
    assert e.value.info["failed_column"] == 1


@pytest.mark.parametrize("m", [100, 300, 1000, 2085])
def test_triangular_solves(ctx, m):
    C = synth.gen_X(m, 0, m, 9)
    T, A, (P, dT, dA, W), _ = _build(ctx, C, G, 1.0, 1e-6, 1e-8)
    rng = np.random.default_rng(m)
    for which, F in ((0, T), (1, A)):
        for trans in (False, True):
            b = rng.standard_normal(m)
            x = host(ctx.precond_solve(P, dT, dA, W, which, trans, dev(b)))
            ref = sla.solve_triangular(F, b, lower=False, trans="T" if trans else "N")
            assert rel_l2(x, ref) <= 1e-10


def _fit_gpu(ctx, X, y, C, kernel, sigma, lam, iters, jitter=1e-8):
    m = C.shape[0]
    alpha, info = ctx.fit(dev(X), dev(y), dev(C), kernel, sigma, lam, iters, zeros(m), jitter)
    return host(alpha), info


@pytest.mark.parametrize("kernel", [G, L])
def test_fit_tiny_config(ctx, kernel):
    """BASELINE.json configs[0]: n=2000, d=8, m=100, sigma=1, lambda=1e-6, 10 iterations."""
    cfg, X, y, C = synth.make_problem("tiny")
    ref = oracle.fit(X, y, C, kernel, cfg.sigma, cfg.lam, cfg.iters)
    alpha, info = _fit_gpu(ctx, X, y, C, kernel, cfg.sigma, cfg.lam, cfg.iters)
    assert info["iters_run"] == cfg.iters
    assert rel_l2(alpha, ref) <= 1e-3
    Xs = synth.gen_X(cfg.seed, 0, 1000, cfg.d, stream=synth.STREAM_XTEST)
    f_ref = oracle.predict(Xs, C, ref, kernel, cfg.sigma)
    f = host(ctx.predict(dev(Xs), dev(C), dev(alpha), kernel, cfg.sigma, zeros(1000)))
    assert rel_l2(f, f_ref) <= 1e-3


@pytest.mark.parametrize("name,n,m", [("msd", 6000, 600), ("higgs", 8000, 800),
                                      ("taxi", 10000, 1000), ("timit", 3000, 500)])
def test_fit_reduced_configs(ctx, name, n, m):
    """Config shapes (d, sigma, lambda, t of Table 3) on a row prefix with fewer centers."""
    cfg, X, y, C = synth.make_problem(name, n=n, m=m)
    ref = oracle.fit(X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    alpha, info = _fit_gpu(ctx, X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    assert rel_l2(alpha, ref) <= 1e-3
    Xs = synth.gen_X(cfg.seed, 0, 2000, cfg.d, stream=synth.STREAM_XTEST)
    f = host(ctx.predict(dev(Xs), dev(C), dev(alpha), G, cfg.sigma, zeros(2000)))
    assert rel_l2(f, oracle.predict(Xs, C, ref, G, cfg.sigma)) <= 1e-3


def test_fit_C_equals_X_identity(ctx):
    """north_star identity: m = n, C = X -> one CG step gives (Knn + n lam I)^-1 y."""
    rng = np.random.default_rng(3)
    n, d, sigma, lam = 200, 8, 1.0, 1e-3   # SURVEY.md E3 setting (Knn well conditioned)
    X = rng.standard_normal((n, d)).astype(np.float32)
    y = np.sin(X[:, 0]).astype(np.float32)
    Knn = oracle.kernel_block(X, X, G, sigma)
    direct = np.linalg.solve(Knn + n * lam * np.eye(n), y.astype(np.float64))
    alpha, _ = _fit_gpu(ctx, X, y, X.copy(), G, sigma, lam, 1, jitter=0.0)
    assert rel_l2(alpha, direct) <= 1e-3


def test_fit_scalar_closed_form(ctx):
    X = np.array([[0.2, 0.1]], dtype=np.float32)
    y = np.array([2.5], dtype=np.float32)
    alpha, info = _fit_gpu(ctx, X, y, X.copy(), G, 1.0, 0.5, 4, jitter=0.0)
    assert abs(alpha[0] - 2.5 / 1.5) <= 1e-6 * 2.5
    assert 1 <= info["iters_run"] <= 4


def test_fit_zero_iterations_and_zero_rhs(ctx):
    cfg, X, y, C = synth.make_problem("tiny")
    alpha, info = _fit_gpu(ctx, X, y, C, G, 1.0, 1e-6, 0)
    assert np.all(alpha == 0.0)
    alpha, info = _fit_gpu(ctx, X, np.zeros_like(y), C, G, 1.0, 1e-6, 5)
    assert np.all(alpha == 0.0) and info["iters_run"] == 0


def test_fit_many_iterations_equals_eq5(ctx):
    """t >> m: GPU alpha solves Eq. (5) to the product's precision."""
    rng = np.random.default_rng(11)
    n, m, d, sigma, lam, delta = 2000, 40, 5, 1.0, 1e-4, 1e-8
    X = rng.standard_normal((n, d)).astype(np.float32)
    C = X[rng.choice(n, m, replace=False)]
    y = np.sin(X.sum(1)).astype(np.float32)
    Knm = oracle.kernel_block(X, C, G, sigma)
    Kmm = oracle.kmm(C, G, sigma) + delta * np.eye(m)
    direct = np.linalg.solve(Knm.T @ Knm + lam * n * Kmm, Knm.T @ y.astype(np.float64))
    alpha, _ = _fit_gpu(ctx, X, y, C, G, sigma, lam, 3 * m, jitter=delta)
    assert rel_l2(alpha, direct) <= 1e-3


@pytest.mark.parametrize("m,k", [(300, 5), (1000, 16), (2085, 21)])
def test_triangular_solves_multi_column(ctx, m, k):
    """Multi-column solve (multi-output fits): every column equals SciPy's solve."""
    from paper_2006_10350_b200 import binding  # noqa: F401
    C = synth.gen_X(m + 1, 0, m, 9)
    T, A, (P, dT, dA, W), _ = _build(ctx, C, G, 1.0, 1e-6, 1e-8)
    rng = np.random.default_rng(m + k)
    for which, F in ((0, T), (1, A)):
        for trans in (False, True):
            B = rng.standard_normal((k, m))  # column-major [k][m]
            Xd = dev(B.copy())
            ctx.precond_solve_multi(P, dT, dA, W, which, trans, Xd)
            ref = sla.solve_triangular(F, B.T, lower=False, trans="T" if trans else "N")
            assert rel_l2(host(Xd).T, ref) <= 1e-10


@pytest.mark.parametrize("m,d", [(3000, 28), (2999, 9), (4352, 90)])
def test_preconditioner_schedules_agree(lib, m, d):
    """The GEMM variants (TMA-fed producer-warp kernel 5 / cp.async kernel 2) and the
    lookahead schedule (next panel on a high-priority stream, bulk trailing update on a
    low-priority one) compute every factor entry with the same k order, so for a given outer
    blocking the factors are bitwise identical; every schedule matches the oracle at fp64
    level.  m = 2999: odd ld (no TMA maps, fallback); outer block 1 x 128 makes the lookahead
    run over many panels (a different blocking: a different fp64 summation association)."""
    from paper_2006_10350_b200 import binding
    C = synth.gen_X(m + 7, 0, m, d)
    To, Ao = oracle.preconditioner(C, G, 3.0, 1e-6, 1e-8)
    ref = {}
    for gemm_v, la, outer in [(2, 0, 8), (5, 0, 8), (5, 1, 8), (2, 0, 1), (5, 1, 1), (2, 1, 1)]:
        c = binding.Context(0)
        try:
            c.set_option(binding.OPT_GEMM_WARPS, gemm_v)
            c.set_option(binding.OPT_LOOKAHEAD, la)
            c.set_option(binding.OPT_POTRF_OUTER, outer)
            T, A, _, info = _build(c, C, G, 3.0, 1e-6, 1e-8)
        finally:
            c.close()
        assert info["failed_factor"] == -1
        assert np.max(np.abs(T - To)) <= 1e-9 * max(1.0, np.max(np.abs(To)))
        assert np.max(np.abs(A - Ao)) <= 1e-8 * max(1.0, np.max(np.abs(Ao)))
        if outer in ref:
            assert np.array_equal(T, ref[outer][0]) and np.array_equal(A, ref[outer][1]), \
                (gemm_v, la, outer)
        else:
            ref[outer] = (T, A)


def test_fit_nonfinite_target_reports_failed_iter(ctx):
    """Reading c9: a NaN target makes the RHS and p^T A p non-finite in the first iteration;
    the device-side breakdown test stops CG and the call returns ENONFINITE with
    failed_iter = 1 (never a silently NaN alpha)."""
    from paper_2006_10350_b200 import binding
    cfg, X, y, C = synth.make_problem("tiny")
    y = y.copy()
    y[123] = np.nan
    with pytest.raises(binding.FalkonError) as ei:
        _fit_gpu(ctx, X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    assert ei.value.code == 3  # FALKON_ENONFINITE
    assert ei.value.info["failed_iter"] == 1
    # the context stays usable afterwards
    alpha, info = _fit_gpu(ctx, X, np.nan_to_num(y), C, G, cfg.sigma, cfg.lam, 2)
    assert np.all(np.isfinite(alpha)) and info["iters_run"] == 2


@pytest.mark.parametrize("name,n,m,expect", [("taxi", 8000, 600, 1), ("tiny", None, None, 1),
                                             ("higgs", 8000, 600, 2), ("msd", 4000, 500, 2)])
def test_fit_precise_path_choice(ctx, name, n, m, expect):
    """Reading d3 (FALKON_OPT_FIT_PRECISE): Gaussian fits whose mean scaled centre norm
    ||c~||^2/2 exceeds 4 at d <= 32 (TAXI: 6.5, tiny: 5.8) run on the SIMT kernels; HIGGS
    (1.4) and MSD (d = 90) keep the tensor kernel.  Reported in falkon_fit_info.product_path."""
    from paper_2006_10350_b200 import binding
    cfg, X, y, C = synth.make_problem(name, n=n, m=m)
    ref = oracle.fit(X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    alpha, info = _fit_gpu(ctx, X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    assert info["product_path"] == expect
    assert rel_l2(alpha, ref) <= 1e-3
    ctx.set_option(binding.OPT_FIT_PRECISE, 0)
    try:
        _, info0 = _fit_gpu(ctx, X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    finally:
        ctx.set_option(binding.OPT_FIT_PRECISE, 1)
    assert info0["product_path"] == 2
