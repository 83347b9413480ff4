"""GPU parity of the 2-CTA-cluster tensor kernels (Q boxes multicast across the cluster,
FALKON_OPT_TC_CLUSTER = 2): same bar as the single-CTA path (north_star: Knm^T(Knm v)
rel-L2 <= 1e-4 vs the fp64 oracle, fits <= 1e-3), odd P-tile counts (the cluster's padding
CTA), both passes, the resident (d16 <= 192) and streaming (d = 440) kernels, and the
single-evaluation strip on top of clusters."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = pytest.mark.gpu
G = oracle.GAUSSIAN


def _problem(n, m, d, seed):
    X = synth.gen_X(seed, 0, n, d).astype(np.float32)
    C = np.ascontiguousarray(X[synth.center_indices(seed, n, m)])
    v = synth.gen_vec(seed, m).astype(np.float64)
    return X, C, v


@pytest.fixture()
def cl_ctx(lib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2006_10350_b200 import binding
    c = binding.Context(device=0)
    c.set_option(binding.OPT_TC_CLUSTER, 2)
    yield c
    c.close()


SHAPES = [
    (1200, 300, 90, 7.0),      # 10 x 3 P tiles (pass A even, pass B odd -> padding CTA)
    (3001, 517, 28, 3.8),      # ragged, 24 x 5 tiles
    (129, 5, 33, 4.0),         # 2 x 1 tiles: pass B is one real CTA + its padding partner
    (700, 250, 440, 14.5),     # streaming-P kernel
    (600, 200, 330, 12.0),     # streaming, 32-aligned segment (332 -> 352) ends mid-box pair
    (20000, 3000, 90, 7.0),    # several waves
]


@pytest.mark.parametrize("n,m,d,sigma", SHAPES)
def test_cluster_product_parity(cl_ctx, n, m, d, sigma):
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(n, m, d, seed=n + 3 * m + d)
    ref = oracle.knm_t_knm_vec(X, C, v, G, sigma)
    for se in (binding.SINGLE_EVAL_OFF, binding.SINGLE_EVAL_ON):
        cl_ctx.set_option(binding.OPT_SINGLE_EVAL, se)
        u = cl_ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m))
        assert rel_l2(host(u), ref) <= 1e-4, se
    w_ref = oracle.knm_vec(X, C, v, G, sigma)
    w = cl_ctx.kernel_vec(dev(X), dev(C), dev(v), G, sigma, zeros(n))
    assert rel_l2(host(w), w_ref) <= 1e-4


def test_cluster_matches_single_cta(cl_ctx):
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(20000, 3000, 90, seed=5)
    dX, dC, dv = dev(X), dev(C), dev(v)
    u2 = host(cl_ctx.knm_matvec(dX, dC, dv, G, 7.0, zeros(3000)))
    assert np.array_equal(u2, host(cl_ctx.knm_matvec(dX, dC, dv, G, 7.0, zeros(3000))))
    cl_ctx.set_option(binding.OPT_TC_CLUSTER, 1)
    u1 = host(cl_ctx.knm_matvec(dX, dC, dv, G, 7.0, zeros(3000)))
    # identical per-CTA arithmetic; only the fp64 order of the per-split partials may differ
    assert rel_l2(u2, u1) <= 1e-12


def test_cluster_fit_parity(cl_ctx):
    X, C, _ = _problem(9000, 400, 90, seed=9)
    y = synth.gen_y(1, X, 0)
    a_ref = oracle.fit(X, y, C, G, 7.0, 2e-6, 20)
    a, _ = cl_ctx.fit(dev(X), dev(y), dev(C), G, 7.0, 2e-6, 20, zeros(400))
    assert rel_l2(host(a), a_ref) <= 1e-3
