"""GPU parity of the fused products (rows a1-a6 of SURVEY.md §8(a)) against the oracle.

Bar (north_star): Knm^T(Knm v) relative L2 error <= 1e-4 against the fp64 oracle on the
same seeded inputs.  The one-sided products (Knm v, Knm^T w) are held to the same bar.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = pytest.mark.gpu
TOL = 1e-4
G, L = oracle.GAUSSIAN, oracle.LAPLACIAN


def _problem(n, m, d, seed, scale=1.0):
    X = synth.gen_X(seed, 0, n, d) * np.float32(scale)
    if m <= n:
        C = X[synth.center_indices(seed, n, m)]
    else:  # more centers than rows: independent draws (C need not be a subset of X)
        C = synth.gen_X(seed + 1, 0, m, d) * np.float32(scale)
    v = synth.gen_vec(seed, m).astype(np.float64)
    return X.astype(np.float32), np.ascontiguousarray(C), v


# shapes span several tiles and ragged tails of both kernels (SIMT small-d, generic d > 32)
SHAPES = [
    (2000, 100, 8, 1.0),      # tiny config (BASELINE.json configs[0])
    (3001, 517, 9, 1.0),      # TAXI-like d, ragged
    (2500, 333, 28, 3.8),     # HIGGS-like d
    (1537, 129, 1, 0.7),      # d = 1
    (777, 1000, 13, 2.0),     # m > n
    (1200, 300, 90, 7.0),     # MSD-like d (tensor path when enabled)
    (700, 250, 440, 14.5),    # TIMIT-like d
    (500, 70, 33, 4.0),       # just above the small-d limit
]


@pytest.mark.parametrize("kernel", [G, L])
@pytest.mark.parametrize("n,m,d,sigma", SHAPES)
def test_knm_matvec_parity(ctx, kernel, n, m, d, sigma):
    X, C, v = _problem(n, m, d, seed=n + m + d)
    ref = oracle.knm_t_knm_vec(X, C, v, kernel, sigma)
    u = ctx.knm_matvec(dev(X), dev(C), dev(v), kernel, sigma, zeros(m))
    assert rel_l2(host(u), ref) <= TOL


@pytest.mark.parametrize("kernel", [G, L])
@pytest.mark.parametrize("n,m,d,sigma", SHAPES[:6])
def test_one_sided_parity(ctx, kernel, n, m, d, sigma):
    X, C, v = _problem(n, m, d, seed=3 * n + m + d)
    w_ref = oracle.knm_vec(X, C, v, kernel, sigma)
    w = ctx.kernel_vec(dev(X), dev(C), dev(v), kernel, sigma, zeros(n))
    assert rel_l2(host(w), w_ref) <= TOL
    wr = np.random.default_rng(n).standard_normal(n)
    u_ref = oracle.knm_t_vec(X, C, wr, kernel, sigma)
    u = ctx.kernel_tvec(dev(X), dev(C), dev(wr), kernel, sigma, zeros(m))
    assert rel_l2(host(u), u_ref) <= TOL


def test_host_pointer_path_matches_device_path(ctx):
    X, C, v = _problem(4000, 300, 9, seed=5)
    ud = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 1.0, zeros(300)))
    uh = np.zeros(300)
    ctx.knm_matvec(X, C, v, G, 1.0, uh)
    assert np.array_equal(ud, uh)


@pytest.mark.parametrize("pinned", [True, False])
def test_host_x_pipelined_path(ctx, pinned):
    """Host X on the tensor path (n >= 8192): rows go up in 8 chunks on a copy stream and each
    chunk is packed + run through pass A as it lands.  Same result as the device path up to the
    fp64 order of per-split partials, and the oracle bar."""
    import torch
    X, C, v = _problem(30001, 1200, 90, seed=15)
    ud = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 7.0, zeros(1200)))
    Xh = torch.from_numpy(X)
    if pinned:
        Xh = Xh.pin_memory()
    uh = np.zeros(1200)
    ctx.knm_matvec(Xh, C, v, G, 7.0, uh)
    assert rel_l2(uh, ud) <= 1e-12
    assert rel_l2(uh, oracle.knm_t_knm_vec(X, C, v, G, 7.0)) <= TOL
    uh2 = np.zeros(1200)
    ctx.knm_matvec(Xh, C, v, G, 7.0, uh2)  # deterministic
    assert np.array_equal(uh, uh2)


def test_deterministic_bitwise(ctx):
    X, C, v = _problem(5000, 700, 28, seed=6)
    a = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 3.8, zeros(700)))
    b = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 3.8, zeros(700)))
    assert np.array_equal(a, b)


def test_zero_vector_and_unit_vectors(ctx):
    X, C, _ = _problem(1000, 50, 9, seed=7)
    u = host(ctx.knm_matvec(dev(X), dev(C), dev(np.zeros(50)), G, 1.0, zeros(50)))
    assert np.all(u == 0.0)
    e = np.zeros(1000)
    e[17] = 1.0
    row = host(ctx.kernel_tvec(dev(X), dev(C), dev(e), G, 1.0, zeros(50)))
    ref = oracle.kernel_block(X[17:18], C, G, 1.0)[0]
    assert rel_l2(row, ref) <= 1e-5


def test_empty_rank_contributes_zero(ctx):
    X = np.zeros((0, 9), np.float32)
    C = synth.gen_X(1, 0, 40, 9)
    u = host(ctx.knm_matvec(dev(X), dev(C), dev(np.ones(40)), G, 1.0, zeros(40)))
    assert np.all(u == 0.0)


def test_single_point(ctx):
    X = synth.gen_X(2, 0, 1, 5)
    C = X.copy()
    u = host(ctx.knm_matvec(dev(X), dev(C), dev(np.array([2.5])), G, 1.0, zeros(1)))
    assert abs(u[0] - 2.5) <= 1e-6


def test_sigma_infinity_closed_form(ctx):
    """sigma -> inf: K == 1 in fp32, u = n * sum(v) (SURVEY.md §8(c) pins), long sums."""
    n, m = 200_000, 64
    X, C, v = _problem(n, m, 9, seed=8)
    v = np.abs(v)
    u = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 1e5, zeros(m)))
    assert np.max(np.abs(u - n * v.sum())) <= 1e-6 * n * v.sum()


def test_translation_invariance(ctx):
    """Shifting X and C by a large common offset (SPEC S:523 flavour) leaves the product
    unchanged: centring removes the norm-expansion cancellation."""
    X, C, v = _problem(3000, 200, 28, seed=9)
    off = np.float32(100.0)
    Xs, Cs = X + off, C + off
    ref = oracle.knm_t_knm_vec(Xs, Cs, v, G, 3.8)
    u = host(ctx.knm_matvec(dev(Xs), dev(Cs), dev(v), G, 3.8, zeros(200)))
    assert rel_l2(u, ref) <= TOL


TC_SHAPES = [
    (1200, 300, 90, 7.0),     # MSD-like
    (4100, 700, 90, 7.0),     # several P tiles and Q tiles, ragged
    (100, 40, 90, 7.0),       # smaller than one tile on both sides
    (900, 513, 33, 4.0),      # d16 = 48
    (640, 260, 186, 10.0),    # largest d of the resident-A tensor kernel (d16 = 192)
    (3000, 2000, 28, 3.8),    # HIGGS d forced onto tensor cores
    (1500, 700, 440, 14.5),   # TIMIT d: streaming-P tensor kernel (64-aligned segments)
    (300, 90, 250, 10.0),     # streaming kernel, sub-tile sizes
]


@pytest.mark.parametrize("n,m,d,sigma", TC_SHAPES)
def test_tensor_path_parity(ctx, n, m, d, sigma):
    """tcgen05 fp16x3 cross-term path (forced) against the oracle, product and one-sided."""
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(n, m, d, seed=7 * n + m + d)
    ctx.set_option(binding.OPT_PATH, binding.PATH_TENSOR)
    try:
        u = ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m))
        w = ctx.kernel_vec(dev(X), dev(C), dev(v), G, sigma, zeros(n))
    finally:
        ctx.set_option(binding.OPT_PATH, binding.PATH_AUTO)
    assert rel_l2(host(w), oracle.knm_vec(X, C, v, G, sigma)) <= TOL
    assert rel_l2(host(u), oracle.knm_t_knm_vec(X, C, v, G, sigma)) <= TOL


def test_tensor_and_simt_paths_agree(ctx):
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(20000, 3000, 90, seed=12)
    out = {}
    for path in (binding.PATH_SIMT, binding.PATH_TENSOR):
        ctx.set_option(binding.OPT_PATH, path)
        out[path] = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 7.0, zeros(3000)))
    ctx.set_option(binding.OPT_PATH, binding.PATH_AUTO)
    assert rel_l2(out[binding.PATH_TENSOR], out[binding.PATH_SIMT]) <= TOL


@pytest.mark.parametrize("n,m,d,sigma", [s for s in SHAPES if s[2] <= 33])
def test_simt_path_parity(ctx, n, m, d, sigma):
    """FP32/MUFU SIMT kernels forced (they serve the Laplacian kernel and d <= 8 by default)."""
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(n, m, d, seed=11 * n + m + d)
    ctx.set_option(binding.OPT_PATH, binding.PATH_SIMT)
    try:
        u = ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(m))
    finally:
        ctx.set_option(binding.OPT_PATH, binding.PATH_AUTO)
    assert rel_l2(host(u), oracle.knm_t_knm_vec(X, C, v, G, sigma)) <= TOL


def test_nccl_collective_path_single_rank():
    """A 1-rank NCCL communicator routes every m-vector through ncclAllReduce (dlopen'ed
    libnccl, ncclCommInitRank, stream-ordered allreduce): results must equal the no-NCCL
    context bit for bit (allreduce over one rank is the identity)."""
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(6000, 700, 28, seed=21)
    y = synth.gen_y(3, X, 0)
    plain = binding.Context(0)
    coll = binding.Context(0, rank=0, world=1, unique_id=binding.get_unique_id())
    try:
        outs = []
        for c in (plain, coll):
            u = host(c.knm_matvec(dev(X), dev(C), dev(v), G, 3.8, zeros(700)))
            a, info = c.fit(dev(X), dev(y), dev(C), G, 3.8, 1e-6, 5, zeros(700))
            outs.append((u, host(a)))
        assert np.array_equal(outs[0][0], outs[1][0])
        assert np.array_equal(outs[0][1], outs[1][1])
        t = coll.timings()
        assert t["allreduce"][1] > 0  # the collective was issued
    finally:
        plain.close()
        coll.close()


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_exp_offload_modes_parity(ctx, mode):
    """exp2 evaluated on the FMA pipe (degree-5 polynomial, FALKON_OPT_EXP_OFFLOAD) for none,
    all, 1/4 or 1/2 of the entries: same 1e-4 product bar, including entries far below 2^-126
    (sigma = 0.6 at d = 28: typical exponents ~ -110; the polynomial path clamps at -126)."""
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(3001, 517, 28, seed=31)
    ctx.set_option(binding.OPT_EXP_OFFLOAD, mode)
    try:
        for sigma in (3.8, 0.6):
            u = ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(517))
            assert rel_l2(host(u), oracle.knm_t_knm_vec(X, C, v, G, sigma)) <= TOL, sigma
    finally:
        ctx.set_option(binding.OPT_EXP_OFFLOAD, 0)


@pytest.mark.parametrize("accum_f64,tol", [(1, 1e-12), (0, 1e-7)])
@pytest.mark.parametrize("d,sigma", [(90, 7.0), (9, 1.0), (8, 1.0)])
def test_sequential_shards_sum_to_full_product(ctx, accum_f64, tol, d, sigma):
    """the row-sharded product is the sum of per-shard products (run
    here one after another on one device through the C ABI, as G ranks would).  With fp64
    contractions (ACCUM_F64) the shard results differ from the unsharded product only in fp64
    summation order (1e-12); the fp32 path's per-tile fp32 partial sums group the rows by
    shard-relative tiles, so it agrees to fp32-partial-sum level."""
    from paper_2006_10350_b200 import binding, parallel
    X, C, v = _problem(20_011, 900, d, seed=31)
    ctx.set_option(binding.OPT_ACCUM_F64, accum_f64)
    try:
        full = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, sigma, zeros(900)))
        for world in (2, 3, 8):
            acc = np.zeros(900)
            for r in range(world):
                lo, hi = parallel.shard_range(X.shape[0], world, r)
                acc += host(ctx.knm_matvec(dev(X[lo:hi]), dev(C), dev(v), G, sigma, zeros(900)))
            assert rel_l2(acc, full) <= tol, world
    finally:
        ctx.set_option(binding.OPT_ACCUM_F64, 0)


def test_tensor_range_guard_falls_back_to_simt(ctx):
    """coordinates or folded biases beyond the fp16 range of the tensor path's
    hi/lo split would turn whole rows into NaN.  The packing kernel flags them and the product
    runs on the fp32 SIMT kernels instead: finite, and bit-identical to the forced SIMT path."""
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(3000, 400, 90, seed=32, scale=400.0)  # ||x~||^2 ~ 2e7 >> fp16 max
    u = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 1.0, zeros(400)))
    ctx.set_option(binding.OPT_PATH, binding.PATH_SIMT)
    try:
        us = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 1.0, zeros(400)))
    finally:
        ctx.set_option(binding.OPT_PATH, binding.PATH_AUTO)
    assert np.all(np.isfinite(u))
    assert np.array_equal(u, us)


def test_ts_variant_with_multi_vector_and_strip(ctx):
    """with FALKON_TC_TS=1 the 192-row TS tensor maps must only feed the TS kernel;
    the multi-vector (kv = 16) and single-evaluation kernels keep 256-row Q boxes."""
    import os
    from paper_2006_10350_b200 import binding
    X, C, v = _problem(4000, 600, 90, seed=33)
    V = np.random.default_rng(3).standard_normal((600, 16))
    ref_u = oracle.knm_t_knm_vec(X, C, v, G, 7.0)
    os.environ["FALKON_TC_TS"] = "1"
    try:
        u = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 7.0, zeros(600)))
        U = host(ctx.knm_matmat(dev(X), dev(C), dev(V), G, 7.0, zeros(600 * 16).reshape(600, 16)))
        ctx.set_option(binding.OPT_SINGLE_EVAL, 1)
        us = host(ctx.knm_matvec(dev(X), dev(C), dev(v), G, 7.0, zeros(600)))
    finally:
        del os.environ["FALKON_TC_TS"]
        ctx.set_option(binding.OPT_SINGLE_EVAL, 2)
    assert rel_l2(u, ref_u) <= TOL
    assert rel_l2(us, ref_u) <= TOL
    for c in (0, 7, 15):
        assert rel_l2(U[:, c], oracle.knm_t_knm_vec(X, C, V[:, c], G, 7.0)) <= TOL


def test_binding_rejects_wrong_sizes_and_devices(ctx):
    """the C ABI trusts sizes, so the binding checks them (a short output would be
    written past its end)."""
    X, C, v = _problem(500, 50, 9, seed=34)
    with pytest.raises(ValueError):
        ctx.knm_matvec(dev(X), dev(C), dev(v), G, 1.0, zeros(49))
    with pytest.raises(ValueError):
        ctx.knm_matvec(dev(X), dev(C), dev(v[:40]), G, 1.0, zeros(50))
    with pytest.raises(ValueError):
        ctx.kernel_vec(dev(X), dev(C), dev(v), G, 1.0, np.zeros(499))
    with pytest.raises(ValueError):
        ctx.fit(dev(X), dev(np.zeros(499, np.float32)), dev(C), G, 1.0, 1e-3, 2, zeros(50))


def test_stuck_pipeline_traps_and_reports_ecuda():
    """A tcgen05 pipeline wait that never completes must not hang the GPU: mbar_wait_safe traps
    after ~4 s of clock64 time, the kernel aborts, and the library call returns FALKON_ECUDA
    (the CUDA context is then unusable - a sticky error - so this runs in a subprocess).
    Fault injected with the diagnostic FALKON_TC_MODE=12 (a stage is never filled)."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2006_10350_b200 import binding
ctx = binding.Context(0)
X = np.random.default_rng(0).standard_normal((2000, 90)).astype(np.float32)
C = X[:300].copy()
u = np.zeros(300)
try:
    ctx.knm_matvec(X, C, np.ones(300), binding.GAUSSIAN, 7.0, u)
    print("NO-ERROR")
except binding.FalkonError as e:
    print("CODE", e.code, str(e)[:200])
'''
    env = dict(os.environ, FALKON_TC_MODE="12")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                       env=env, cwd=root)
    assert "CODE 5" in r.stdout, (r.stdout, r.stderr[-1000:])
