"""GPU parity of the single-evaluation product.

Pass A over a strip of rows also stores its kernel values k(x_i, c_j) (fp32, row-major) and a
streaming GEMV reads them back for u += strip^T w, so every entry is evaluated once instead of
twice.  Same bar as the two-pass product (north_star): Knm^T(Knm v) rel-L2 <= 1e-4 against the
fp64 oracle, fits <= 1e-3.  Strips are forced small (64 MiB, the minimum) so that several
strips, a ragged last strip and centre counts that are not a multiple of 4 are exercised.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = pytest.mark.gpu
G = oracle.GAUSSIAN
MiB = 1 << 20


def _problem(n, m, d, seed):
    X = synth.gen_X(seed, 0, n, d)
    C = np.ascontiguousarray(X[synth.center_indices(seed, n, m)])
    v = synth.gen_vec(seed, m).astype(np.float64)
    return X.astype(np.float32), C, v


@pytest.fixture()
def se_ctx(lib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2006_10350_b200 import binding
    c = binding.Context(device=0)
    c.set_option(binding.OPT_SINGLE_EVAL, binding.SINGLE_EVAL_ON)
    c.set_option(binding.OPT_STRIP_BYTES, 64 * MiB)
    yield c
    c.close()


# (n, m, d, sigma): rows per 64 MiB strip = 128 * floor(2^26 / (512 m))
SHAPES = [
    (3001, 517, 28, 3.8),      # one strip, resident-P kernel (16 epilogue warps), m % 4 != 0
    (70001, 517, 9, 1.0),      # 3 strips (32384 rows each) + ragged tail, TAXI-like d
    (5000, 700, 90, 7.0),      # MSD-like d
    (20000, 2100, 440, 14.5),  # 3 strips (7936 rows), streaming-P kernel, TIMIT-like d
    (1500, 300, 250, 10.0),    # streaming kernel, partial tiles on both sides
    (129, 5, 33, 4.0),         # sub-tile sizes
]


@pytest.mark.parametrize("n,m,d,sigma", SHAPES)
def test_single_eval_product_parity(se_ctx, n, m, d, sigma):
    X, C, v = _problem(n, m, d, seed=5 * n + m + d)
    ref = oracle.knm_t_knm_vec(X, C, v, G, sigma)
    u = se_ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m))
    assert rel_l2(host(u), ref) <= 1e-4
    t = se_ctx.timings()
    assert t["pass_b"][1] >= 1  # the strip GEMV ran as the second contraction


@pytest.mark.parametrize("n,m,d,sigma", [SHAPES[1], SHAPES[3]])
def test_single_eval_matches_two_pass_and_is_deterministic(se_ctx, n, m, d, sigma):
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(n, m, d, seed=7 * n + d)
    dX, dC, dv = dev(X), dev(C), dev(v)
    u1 = host(se_ctx.knm_matvec(dX, dC, dv, G, sigma, zeros(m)))
    u2 = host(se_ctx.knm_matvec(dX, dC, dv, G, sigma, zeros(m)))
    assert np.array_equal(u1, u2)
    se_ctx.set_option(binding.OPT_SINGLE_EVAL, binding.SINGLE_EVAL_OFF)
    u0 = host(se_ctx.knm_matvec(dX, dC, dv, G, sigma, zeros(m)))
    # same fp32 kernel values, different fp32 summation order of the second contraction
    assert rel_l2(u1, u0) <= 1e-6


def test_single_eval_sigma_inf_closed_form(se_ctx):
    """sigma -> inf: K == 1 exactly in fp32, so u = n (sum_j v_j) 1 (SURVEY.md §8(c) pins);
    all terms positive and equal, the worst case for long fp32 sums in the GEMV."""
    n, m, d = 50001, 1030, 300
    X = synth.gen_X(3, 0, n, d).astype(np.float32)
    C = np.ascontiguousarray(X[synth.center_indices(3, n, m)])
    v = np.abs(synth.gen_vec(3, m)).astype(np.float32).astype(np.float64)
    u = host(se_ctx.knm_matvec(dev(X), dev(C), dev(v), G, 1e5, zeros(m)))
    exact = n * v.sum()
    assert np.max(np.abs(u - exact)) / exact <= 1e-6


@pytest.mark.parametrize("n,m,d,sigma,lam,iters", [
    (6000, 300, 440, 14.5, 5e-9, 5),   # TIMIT-shaped (Table 3 sigma, lambda, t)
    (9000, 400, 90, 7.0, 2e-6, 20),    # MSD-shaped
])
def test_single_eval_fit_parity(se_ctx, n, m, d, sigma, lam, iters):
    X, C, _ = _problem(n, m, d, seed=n + d)
    y = synth.gen_y(1, X, 0).astype(np.float32)
    a_ref = oracle.fit(X, y, C, G, sigma, lam, iters)
    a, info = se_ctx.fit(dev(X), dev(y), dev(C), G, sigma, lam, iters, zeros(m))
    assert rel_l2(host(a), a_ref) <= 1e-3
    Xs = synth.gen_X(77, 0, 2000, d).astype(np.float32)
    f_ref = oracle.predict(Xs, C, a_ref, G, sigma)
    f = se_ctx.predict(dev(Xs), dev(C), a, G, sigma, zeros(2000))
    assert rel_l2(host(f), f_ref) <= 1e-3


def test_single_eval_weighted_gsc_parity(se_ctx, ctx):
    """GSC-Falkon / LogFalkon (Alg. 2) on the single-evaluation product: the strip GEMV applies
    the row weights D of the weighted LinOp Knm^T D Knm.  Same alpha as the two-pass product
    up to the problem's conditioning and the oracle bar.  Shape of test_gpu_gsc's well-posed
    tensor case (alpha moves <= 1e-5 under 6e-8 relative noise on the kernel values)."""
    from oracle import gsc
    n, m, d, sigma = 16_001, 300, 90, 7.0
    X = synth.gen_X(3, 0, n, d)
    y = synth.gen_y(3, X, 0, "cls")
    idx = synth.center_indices(3, n, m)
    C, yC = X[idx].copy(), y[idx].copy()
    mus, its = [1e-3, 1e-4, 1e-5, 1e-6], [4, 4, 4, 8]
    out = []
    for c in (se_ctx, ctx):  # single evaluation forced (one 64 MiB strip) / default two-pass
        a = zeros(m)
        c.gsc_fit(dev(X), dev(y), dev(C), dev(yC), G, sigma, "logistic", mus, its, a)
        out.append(host(a))
    ao = gsc.gsc_falkon(X, y, C, yC, gsc.LOGISTIC, G, sigma, mus, its)
    assert rel_l2(out[0], ao) <= 1e-3
    assert rel_l2(out[0], out[1]) <= 1e-4


@pytest.mark.parametrize("accum_f64", [0, 1])
def test_fused_strip_gemv_variant(ctx, accum_f64):
    """Experimental FALKON_FUSED_GEMV=1: the GEMV of strip s - 1 runs in warps 2-3 of strip s's
    pass-A launch through a bulk-copy ring (two k buffers, so strips are half as long: the
    fp32 path's per-strip partial sums group differently, 1e-7; fp64 contractions 1e-12),
    and the oracle bar."""
    import os
    from paper_2006_10350_b200 import binding
    n, m, d, sigma = 9001, 700, 300, 12.0
    X = synth.gen_X(41, 0, n, d)
    C = X[synth.center_indices(41, n, m)]
    v = synth.gen_vec(41, m).astype(np.float64)
    ctx.set_option(binding.OPT_SINGLE_EVAL, 1)
    ctx.set_option(binding.OPT_STRIP_BYTES, 64 << 20)
    ctx.set_option(binding.OPT_ACCUM_F64, accum_f64)
    try:
        a = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m)))
        os.environ["FALKON_FUSED_GEMV"] = "1"
        try:
            b = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m)))
        finally:
            del os.environ["FALKON_FUSED_GEMV"]
    finally:
        ctx.set_option(binding.OPT_SINGLE_EVAL, 2)
        ctx.set_option(binding.OPT_STRIP_BYTES, 16 << 30)
        ctx.set_option(binding.OPT_ACCUM_F64, 0)
    assert rel_l2(b, a) <= (1e-12 if accum_f64 else 1e-7)
    assert rel_l2(b, oracle.knm_t_knm_vec(X, C, v, G, sigma)) <= 1e-4


@pytest.mark.parametrize("pair", ["0", "1", "2"])
@pytest.mark.parametrize("se,accum_f64", [(0, 0), (1, 0), (1, 1), (0, 1)])
@pytest.mark.parametrize("d,sigma", [(440, 14.5), (90, 7.0)])
def test_cta_pair_variant(ctx, pair, se, accum_f64, d, sigma):
    """CTA-pair MMAs (cta_group::2): default for the streaming kernel (d > 190), opt-in
    (FALKON_TC_PAIR=2) for the resident one; FALKON_TC_PAIR=0 = multicast-only clusters.
    Oracle bar for two-pass and single-evaluation products, fp32 and fp64 contractions."""
    import os
    from paper_2006_10350_b200 import binding
    n, m = 3001, 771
    X = synth.gen_X(43, 0, n, d)
    C = X[synth.center_indices(43, n, m)]
    v = synth.gen_vec(43, m).astype(np.float64)
    ctx.set_option(binding.OPT_SINGLE_EVAL, se)
    ctx.set_option(binding.OPT_ACCUM_F64, accum_f64)
    os.environ["FALKON_TC_PAIR"] = pair
    try:
        u = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m)))
    finally:
        del os.environ["FALKON_TC_PAIR"]
        ctx.set_option(binding.OPT_SINGLE_EVAL, 2)
        ctx.set_option(binding.OPT_ACCUM_F64, 0)
    assert rel_l2(u, oracle.knm_t_knm_vec(X, C, v, G, sigma)) <= 1e-4


@pytest.mark.parametrize("accum_f64", [0, 1])
@pytest.mark.parametrize("gsm", [1, 16, 147])
def test_split_sm_gemv_variant(ctx, accum_f64, gsm):
    """FALKON_OPT_SE_GEMV_SMS = G > 0: the GEMV of strip s as a persistent grid of G CTAs
    (se_gemv_ldg_kernel, one 768-thread CTA per SM) on a second stream beside pass A of strip s + 1, two
    strip buffers, the last strip's GEMV on the whole GPU.  Deterministic, the serial schedule
    to fp32 regrouping (fp64 contractions: 1e-12) and the oracle bar; 5 strips + ragged tail,
    m not a multiple of the 8-centre groups."""
    from paper_2006_10350_b200 import binding
    n, m, d, sigma = 40001, 1030, 300, 12.0
    X = synth.gen_X(47, 0, n, d)
    C = X[synth.center_indices(47, n, m)]
    v = synth.gen_vec(47, m).astype(np.float64)
    dX, dC, dv = dev(X), dev(C), dev(v)
    ctx.set_option(binding.OPT_SINGLE_EVAL, 1)
    ctx.set_option(binding.OPT_STRIP_BYTES, 64 << 20)
    ctx.set_option(binding.OPT_ACCUM_F64, accum_f64)
    try:
        a = host(ctx.knm_matvec(dX, dC, dv, G, sigma, zeros(m)))
        ctx.set_option(binding.OPT_SE_GEMV_SMS, gsm)
        b1 = host(ctx.knm_matvec(dX, dC, dv, G, sigma, zeros(m)))
        b2 = host(ctx.knm_matvec(dX, dC, dv, G, sigma, zeros(m)))
    finally:
        ctx.set_option(binding.OPT_SE_GEMV_SMS, 0)
        ctx.set_option(binding.OPT_SINGLE_EVAL, 2)
        ctx.set_option(binding.OPT_STRIP_BYTES, 16 << 30)
        ctx.set_option(binding.OPT_ACCUM_F64, 0)
    assert np.array_equal(b1, b2)
    assert rel_l2(b1, a) <= (1e-12 if accum_f64 else 1e-7)
    assert rel_l2(b1, oracle.knm_t_knm_vec(X, C, v, G, sigma)) <= 1e-4


def test_split_sm_gemv_option_range(ctx):
    from paper_2006_10350_b200 import binding
    with pytest.raises(binding.FalkonError):
        ctx.set_option(binding.OPT_SE_GEMV_SMS, -1)
    with pytest.raises(binding.FalkonError):
        ctx.set_option(binding.OPT_SE_GEMV_SMS, 100000)
