"""GPU parity of the fp64-accumulation contractions (FALKON_OPT_ACCUM_F64 = 1).

SURVEY.md §7 hard part 3: carrying v and w in fp64 and accumulating the exact products
k(x, c) * v by DFMA leaves the fp32 rounding of k itself as the only product error.  Bars:
the north_star 1e-4 on the product, and (tighter, as the variant's purpose) a product error
no larger than the fp32 path's on the same inputs; the sigma -> inf closed form (K == 1
exactly in fp32) must then hold to fp64 rounding, not to the 1e-6 of fp32 partial sums.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros
from test_gpu_product import SHAPES, _problem

pytestmark = pytest.mark.gpu
G, L = oracle.GAUSSIAN, oracle.LAPLACIAN


@pytest.fixture(scope="module")
def ctx64(lib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2006_10350_b200 import binding
    c = binding.Context(device=0)
    c.set_option(binding.OPT_ACCUM_F64, 1)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx32(lib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2006_10350_b200 import binding
    c = binding.Context(device=0)
    c.set_option(binding.OPT_ACCUM_F64, 0)
    yield c
    c.close()


def _set_path(c, path):
    from paper_2006_10350_b200 import binding
    c.set_option(binding.OPT_PATH, path)


@pytest.mark.parametrize("path", [0, 1, 2])  # auto, SIMT, tensor
@pytest.mark.parametrize("kernel", [G, L])
@pytest.mark.parametrize("n,m,d,sigma", SHAPES)
def test_knm_matvec_f64_parity(ctx64, ctx32, kernel, path, n, m, d, sigma):
    if path == 2 and kernel == L:
        pytest.skip("Laplacian has no tensor path (reading c7)")
    X, C, v = _problem(n, m, d, seed=n + m + d)
    ref = oracle.knm_t_knm_vec(X, C, v, kernel, sigma)
    _set_path(ctx64, path)
    _set_path(ctx32, path)
    try:
        u64 = host(ctx64.knm_matvec(dev(X), dev(C), dev(v), kernel, sigma, zeros(m)))
        u32 = host(ctx32.knm_matvec(dev(X), dev(C), dev(v), kernel, sigma, zeros(m)))
    finally:
        _set_path(ctx64, 0)
        _set_path(ctx32, 0)
    e64, e32 = rel_l2(u64, ref), rel_l2(u32, ref)
    assert e64 <= 1e-4
    assert e64 <= 1.5 * e32 + 1e-9, (e64, e32)


@pytest.mark.parametrize("kernel", [G, L])
@pytest.mark.parametrize("n,m,d,sigma", SHAPES[:6])
def test_one_sided_f64_parity(ctx64, kernel, n, m, d, sigma):
    X, C, v = _problem(n, m, d, seed=3 * n + m + d)
    w_ref = oracle.knm_vec(X, C, v, kernel, sigma)
    w = ctx64.kernel_vec(dev(X), dev(C), dev(v), kernel, sigma, zeros(n))
    assert rel_l2(host(w), w_ref) <= 1e-5
    wr = np.random.default_rng(n).standard_normal(n)
    u_ref = oracle.knm_t_vec(X, C, wr, kernel, sigma)
    u = ctx64.kernel_tvec(dev(X), dev(C), dev(wr), kernel, sigma, zeros(m))
    assert rel_l2(host(u), u_ref) <= 1e-5


@pytest.mark.parametrize("path", [1, 2])
def test_sigma_infinity_closed_form_f64(ctx64, path):
    """K == 1 exactly (sigma = 1e5), u = n * sum(v): with DFMA accumulation the error is fp64
    rounding of a long positive sum, ~1e-13, not the fp32 1e-6."""
    n, m = 200_000, 64
    X, C, v = _problem(n, m, 9, seed=8)
    v = np.abs(v)
    _set_path(ctx64, path)
    try:
        u = host(ctx64.knm_matvec(dev(X), dev(C), dev(v), G, 1e5, zeros(m)))
    finally:
        _set_path(ctx64, 0)
    assert np.max(np.abs(u - n * v.sum())) <= 1e-12 * n * v.sum()


def test_single_eval_f64(ctx64):
    """Single-evaluation strip product (k strip + DFMA GEMV over fp64 w) vs the two-pass fp64
    product and the oracle; several strips and a ragged last one; bitwise deterministic."""
    from paper_2006_10350_b200 import binding
    n, m, d, sigma = 9000, 700, 300, 12.0
    X, C, v = _problem(n, m, d, seed=21)
    ref = oracle.knm_t_knm_vec(X, C, v, G, sigma)
    ctx64.set_option(binding.OPT_SINGLE_EVAL, 0)
    two = host(ctx64.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m)))
    ctx64.set_option(binding.OPT_SINGLE_EVAL, 1)
    ctx64.set_option(binding.OPT_STRIP_BYTES, 64 << 20)  # 64 MiB / (4 m) rows: several strips
    try:
        one = host(ctx64.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m)))
        one2 = host(ctx64.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m)))
    finally:
        ctx64.set_option(binding.OPT_SINGLE_EVAL, 2)
        ctx64.set_option(binding.OPT_STRIP_BYTES, 16 << 30)
    # pass B of the two-pass product recomputes k with the operands' roles swapped (the fp32
    # rounding of the three MMA terms may differ by an ulp); the strip reuses pass A's k
    assert rel_l2(one, two) <= 1e-8
    assert rel_l2(one, ref) <= 1e-5
    assert np.array_equal(one, one2)


def test_deterministic_bitwise_f64(ctx64):
    X, C, v = _problem(5000, 700, 28, seed=6)
    a = host(ctx64.knm_matvec(dev(X), dev(C), dev(v), G, 3.8, zeros(700)))
    b = host(ctx64.knm_matvec(dev(X), dev(C), dev(v), G, 3.8, zeros(700)))
    assert np.array_equal(a, b)


@pytest.mark.parametrize("kernel", [G, L])
def test_fit_tiny_f64(ctx64, kernel):
    cfg, X, y, C = synth.make_problem("tiny")
    aref = oracle.fit(X, y, C, kernel, cfg.sigma, cfg.lam, cfg.iters)
    alpha, info = ctx64.fit(dev(X), dev(y), dev(C), kernel, cfg.sigma, cfg.lam, cfg.iters,
                            zeros(cfg.m))
    assert rel_l2(host(alpha), aref) <= 1e-3
    Xs = synth.gen_X(cfg.seed, 0, 1000, cfg.d, stream=synth.STREAM_XTEST)
    f = host(ctx64.predict(dev(Xs), dev(C), alpha, kernel, cfg.sigma, zeros(1000)))
    assert rel_l2(f, oracle.predict(Xs, C, aref, kernel, cfg.sigma)) <= 1e-3


@pytest.mark.parametrize("config,n,m", [("msd", 20000, 1000), ("higgs", 20000, 1000),
                                        ("taxi", 20000, 1000), ("timit", 6000, 800)])
def test_fit_prefix_f64_not_worse(ctx64, ctx32, config, n, m):
    """Config-shaped prefixes: fp64 accumulation meets the 1e-3 bar and is not worse than fp32."""
    cfg, X, y, C = synth.make_problem(config, n=n, m=m)
    aref = oracle.fit(X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    a64, _ = ctx64.fit(dev(X), dev(y), dev(C), G, cfg.sigma, cfg.lam, cfg.iters, zeros(m))
    a32, _ = ctx32.fit(dev(X), dev(y), dev(C), G, cfg.sigma, cfg.lam, cfg.iters, zeros(m))
    e64, e32 = rel_l2(host(a64), aref), rel_l2(host(a32), aref)
    assert e64 <= 1e-3
    assert e64 <= 1.5 * e32 + 1e-9, (e64, e32)


def test_gsc_fit_f64(ctx64):
    """LogFalkon (Alg. 2) with fp64 contractions against the GSC oracle (tiny_log)."""
    from oracle import gsc_oracle as gsc
    g = synth.GSC_CONFIGS["tiny_log"]
    _, X, y, C, yC = synth.make_gsc_problem("tiny_log")
    aref = gsc.gsc_falkon(X, y, C, yC, gsc.LOGISTIC, G, g.sigma, g.mus, g.iters)
    alpha, _ = ctx64.gsc_fit(dev(X), dev(y), dev(C), dev(yC), G, g.sigma, "logistic",
                             list(g.mus), list(g.iters), zeros(g.m))
    assert rel_l2(host(alpha), aref) <= 1e-3
