"""GPU parity of the fp64 product path (FALKON_PATH_F64, csrc/kvp.cu kvp64_kernel; DESIGN.md
reading d4) and of the fit-time rule that selects it (FALKON_OPT_FIT_PRECISE: d <= 32 and
m > 25,000).

Everything on this path is fp64 (coordinates from the fp32 inputs, exponent, exp2,
contractions), so the bar is the fp64 oracle's own rounding level: products 1e-12 relative,
fits 1e-8 on alpha (CG amplifies rounding-level differences of the summation order).
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = pytest.mark.gpu
G, L = oracle.GAUSSIAN, oracle.LAPLACIAN


@pytest.fixture()
def f64(ctx):
    from paper_2006_10350_b200 import binding
    ctx.set_option(binding.OPT_PATH, binding.PATH_F64)
    yield ctx
    ctx.set_option(binding.OPT_PATH, binding.PATH_AUTO)


@pytest.mark.parametrize("n,m,d,kernel,sigma", [
    (3001, 517, 9, G, 1.0), (4097, 300, 28, G, 3.8), (2000, 257, 90, G, 7.0),
    (1500, 130, 440, G, 14.5), (2999, 301, 28, L, 3.8), (129, 5, 3, G, 0.7), (777, 77, 33, L, 5.0),
])
def test_f64_product_parity(f64, n, m, d, kernel, sigma):
    X = synth.gen_X(n + d, 0, n, d)
    C = np.ascontiguousarray(X[synth.center_indices(n + d, n, m)])
    v = synth.gen_vec(n + d, m).astype(np.float64)
    ref = oracle.knm_t_knm_vec(X, C, v, kernel, sigma)
    u = host(f64.knm_matvec(dev(X), dev(C), dev(v), kernel, sigma, zeros(m)))
    assert rel_l2(u, ref) <= 1e-12


def test_f64_one_sided_and_predict(f64):
    n, m, d, sigma = 5001, 403, 28, 3.8
    X = synth.gen_X(9, 0, n, d)
    C = np.ascontiguousarray(X[synth.center_indices(9, n, m)])
    v = synth.gen_vec(9, m).astype(np.float64)
    w = host(f64.kernel_vec(dev(X), dev(C), dev(v), G, sigma, zeros(n)))
    assert rel_l2(w, oracle.knm_vec(X, C, v, G, sigma)) <= 1e-12


def test_f64_fit_parity(f64):
    n, m, d, sigma, lam, iters = 20000, 1200, 28, 3.8, 3e-8, 10
    X = synth.gen_X(n + d, 0, n, d)
    y = synth.gen_y(2, X, 0).astype(np.float32)
    C = np.ascontiguousarray(X[synth.center_indices(n + d, n, m)])
    a_ref = oracle.fit(X, y, C, G, sigma, lam, iters)
    a, info = f64.fit(dev(X), dev(y), dev(C), G, sigma, lam, iters, zeros(m))
    assert info["product_path"] == 3
    assert rel_l2(host(a), a_ref) <= 1e-8


def test_fit_rule_selects_f64_for_small_d_large_m(ctx):
    """FIT_PRECISE default: d <= 32 and m > 25,000 -> FALKON_PATH_F64; d > 32 keeps its path."""
    from paper_2006_10350_b200 import binding
    n, m = 30000, 25001
    for d, want in ((9, binding.PATH_F64), (40, binding.PATH_TENSOR)):
        X = synth.gen_X(5 + d, 0, n, d)
        y = synth.gen_y(5, X, 0).astype(np.float32)
        C = np.ascontiguousarray(X[synth.center_indices(5 + d, n, m)])
        _, info = ctx.fit(dev(X), dev(y), dev(C), G, 4.0, 1e-6, 1, zeros(m))
        assert info["product_path"] == want, (d, info["product_path"])
    ctx.set_option(binding.OPT_FIT_PRECISE, 0)
    try:
        X = synth.gen_X(14, 0, n, 9)
        y = synth.gen_y(5, X, 0).astype(np.float32)
        C = np.ascontiguousarray(X[synth.center_indices(14, n, m)])
        _, info = ctx.fit(dev(X), dev(y), dev(C), G, 4.0, 1e-6, 1, zeros(m))
        assert info["product_path"] != binding.PATH_F64
    finally:
        ctx.set_option(binding.OPT_FIT_PRECISE, 1)


def test_f64_multi_output_unsupported(f64):
    from paper_2006_10350_b200 import FalkonError
    n, m, d, k = 1000, 100, 9, 8
    X = synth.gen_X(3, 0, n, d)
    C = np.ascontiguousarray(X[:m])
    V = np.ones((m, k))
    with pytest.raises(FalkonError):
        f64.knm_matmat(dev(X), dev(C), dev(V), G, 1.0, zeros((m, k)))
