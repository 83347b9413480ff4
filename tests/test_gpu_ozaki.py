"""GPU parity of the Ozaki-scheme preconditioner GEMMs (FALKON_OPT_OZAKI, csrc/ozaki.cu).

The Cholesky trailing updates run as 36 exact int8 x int8 -> int32 tcgen05 products of
row-scaled 7-bit slices, recombined in fp64.  Bars: the same as the DMMA build against the
fp64 oracle (factors 1e-9 / 1e-8, Cholesky identities 1e-11), agreement with the DMMA build to
~1e-13 relative, determinism, bitwise independence of the schedule (lookahead on / off,
distributed build simulated on one device: every element sees the same k ranges, hence the
same slices and integer sums), ENOTPD, and Falkon fit parity.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = pytest.mark.gpu
G = oracle.GAUSSIAN


def _build(ctx, C, sigma, lam=1e-6, jit=1e-8, kernel=G):
    import torch
    m = C.shape[0]
    P = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    dT, dA = zeros(m), zeros(m)
    W = zeros(ctx.precond_work_elems(m))
    info = ctx.precond_build(dev(C), kernel, sigma, lam, jit, P, dT, dA, W)
    Ph, dTh, dAh = host(P), host(dT), host(dA)
    T = np.triu(Ph, 1) + np.diag(dTh)
    A = (np.tril(Ph, -1) + np.diag(dAh)).T
    return T, A, info


@pytest.fixture()
def oz(ctx):
    from paper_2006_10350_b200 import binding
    ctx.set_option(binding.OPT_OZAKI, 1)  # the default; set explicitly
    yield ctx
    ctx.set_option(binding.OPT_OZAKI, 1)


@pytest.mark.parametrize("m,d,sigma", [(1500, 28, 3.8), (3001, 90, 7.0), (2177, 9, 1.0)])
def test_ozaki_factors_vs_oracle_and_dmma(ctx, m, d, sigma):
    from paper_2006_10350_b200 import binding
    lam, jit = 1e-6, 1e-8
    C = synth.gen_X(m + 3 * d, 0, m, d)
    ctx.set_option(binding.OPT_OZAKI, 0)  # fp64 DMMA reference build
    try:
        T0, A0, _ = _build(ctx, C, sigma, lam, jit)
    finally:
        ctx.set_option(binding.OPT_OZAKI, 1)
    T1, A1, info = _build(ctx, C, sigma, lam, jit)
    T2, A2, _ = _build(ctx, C, sigma, lam, jit)
    assert info["failed_factor"] == -1
    assert np.array_equal(T1, T2) and np.array_equal(A1, A2)  # deterministic
    assert np.max(np.abs(T1 - T0)) <= 1e-12 * np.max(np.abs(T0))
    assert np.max(np.abs(A1 - A0)) <= 1e-11 * np.max(np.abs(A0))
    To, Ao = oracle.preconditioner(C, G, sigma, lam, jit)
    assert np.max(np.abs(T1 - To)) <= 1e-9 * max(1.0, np.max(np.abs(To)))
    assert np.max(np.abs(A1 - Ao)) <= 1e-8 * max(1.0, np.max(np.abs(Ao)))
    K = oracle.kmm(C, G, sigma) + jit * np.eye(m)
    assert np.max(np.abs(T1.T @ T1 - K)) <= 1e-11
    M = T1 @ T1.T / m + lam * np.eye(m)
    assert np.max(np.abs(A1.T @ A1 - M)) <= 1e-11


def test_ozaki_schedule_independent(oz):
    """Lookahead (two streams, one slab each) on / off and the distributed schedule (G = 2
    ranks simulated) give bitwise-identical factors."""
    import torch
    from paper_2006_10350_b200 import binding
    m, d, sigma = 2600, 28, 3.8
    C = synth.gen_X(91, 0, m, d)
    T1, A1, _ = _build(oz, C, sigma)
    oz.set_option(binding.OPT_LOOKAHEAD, 0)
    try:
        T2, A2, _ = _build(oz, C, sigma)
    finally:
        oz.set_option(binding.OPT_LOOKAHEAD, 1)
    assert np.array_equal(T1, T2) and np.array_equal(A1, A2)
    Ps = [torch.zeros((m, m), dtype=torch.float64, device="cuda") for _ in range(2)]
    dTs, dAs = [zeros(m) for _ in range(2)], [zeros(m) for _ in range(2)]
    Ws = [zeros(oz.precond_work_elems(m)) for _ in range(2)]
    oz.precond_build_sim(dev(C), G, sigma, 1e-6, 1e-8, Ps, dTs, dAs, Ws)
    for P, dT, dA in zip(Ps, dTs, dAs):
        Ph = host(P)
        assert np.array_equal(np.triu(Ph, 1) + np.diag(host(dT)), T1)
        assert np.array_equal((np.tril(Ph, -1) + np.diag(host(dA))).T, A1)


def test_ozaki_not_pd(oz):
    from paper_2006_10350_b200 import FalkonError
    m = 1300
    C = np.repeat(synth.gen_X(5, 0, 1, 4), m, axis=0)  # identical centres: Kmm = 1 (rank 1)
    with pytest.raises(FalkonError) as e:
        _build(oz, C, 1.0, jit=0.0)
    assert e.value.info["failed_factor"] == 0


@pytest.mark.parametrize("n,m,d,sigma,lam,iters", [
    (20000, 1500, 28, 3.8, 3e-8, 10),   # HIGGS-shaped
    (12000, 1200, 90, 7.0, 2e-6, 20),   # MSD-shaped
])
def test_ozaki_fit_parity(oz, n, m, d, sigma, lam, iters):
    X = synth.gen_X(n + d, 0, n, d)
    y = synth.gen_y(2, X, 0).astype(np.float32)
    C = np.ascontiguousarray(X[synth.center_indices(n + d, n, m)])
    a_ref = oracle.fit(X, y, C, G, sigma, lam, iters)
    a, _ = oz.fit(dev(X), dev(y), dev(C), G, sigma, lam, iters, zeros(m))
    assert rel_l2(host(a), a_ref) <= 1e-3


def test_ozaki_weighted_lauum_gsc(oz, ctx):
    """GSC-Falkon / LogFalkon (Alg. 2): A is rebuilt per Newton step through the weighted LAUUM
    T D T^T (kscale on the B operand: its own slab); alpha within the oracle bar and 1e-9 of the
    DMMA build."""
    from oracle import gsc
    from paper_2006_10350_b200 import binding
    n, m, d, sigma = 12001, 1400, 28, 3.8
    X = synth.gen_X(17, 0, n, d)
    y = synth.gen_y(17, X, 0, "cls")
    idx = synth.center_indices(17, n, m)
    C, yC = X[idx].copy(), y[idx].copy()
    mus, its = [1e-3, 1e-4], [4, 6]
    a1 = zeros(m)
    oz.gsc_fit(dev(X), dev(y), dev(C), dev(yC), G, sigma, "logistic", mus, its, a1)
    oz.set_option(binding.OPT_OZAKI, 0)
    a0 = zeros(m)
    oz.gsc_fit(dev(X), dev(y), dev(C), dev(yC), G, sigma, "logistic", mus, its, a0)
    oz.set_option(binding.OPT_OZAKI, 1)
    ao = gsc.gsc_falkon(X, y, C, yC, gsc.LOGISTIC, G, sigma, mus, its)
    assert rel_l2(host(a1), ao) <= 1e-3
    assert rel_l2(host(a1), host(a0)) <= 1e-9


def test_ozaki_and_outer_block_options(ctx):
    """FALKON_OPT_OZAKI takes 0 / 1; FALKON_OPT_POTRF_OUTER takes 0 (auto: 16 with Ozaki, 8 with
    DMMA) .. 64; the auto and the explicit 16 build give bitwise-identical factors."""
    from paper_2006_10350_b200 import FalkonError, binding
    for bad in (-1, 2):
        with pytest.raises(FalkonError):
            ctx.set_option(binding.OPT_OZAKI, bad)
    for bad in (-1, 65):
        with pytest.raises(FalkonError):
            ctx.set_option(binding.OPT_POTRF_OUTER, bad)
    C = synth.gen_X(23, 0, 2600, 28)
    try:
        ctx.set_option(binding.OPT_POTRF_OUTER, 0)
        T0, A0, _ = _build(ctx, C, 3.8)
        ctx.set_option(binding.OPT_POTRF_OUTER, 16)
        T1, A1, _ = _build(ctx, C, 3.8)
    finally:
        ctx.set_option(binding.OPT_POTRF_OUTER, 0)
    assert np.array_equal(T0, T1) and np.array_equal(A0, A1)
