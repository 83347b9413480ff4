"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The oracle cannot evaluate a whole n*m product at these sizes in seconds, so each test checks
SAMPLED outputs the oracle computes one by one:
  * w = Knm v on sampled rows (each row: m kernel values),
  * u = Knm^T w on sampled centers, with w the GPU's own full fp64 w (each center: n values),
  * the fused u = Knm^T(Knm v) against the composition of the two checked one-sided passes,
  * the sigma -> inf closed form u = n * sum(v) on the full X.
Tolerance: north_star's 1e-4 relative L2 over the sample.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
G = oracle.GAUSSIAN
TOL = 1e-4


@pytest.fixture(scope="module", params=["msd", "timit", "higgs"])
def full_problem(request):
    cfg = synth.CONFIGS[request.param]
    X = synth.gen_X(cfg.seed, 0, cfg.n, cfg.d)
    C = synth.gen_rows(cfg.seed, synth.STREAM_X, synth.center_indices(cfg.seed, cfg.n, cfg.m), cfg.d)
    v = synth.gen_vec(cfg.seed, cfg.m).astype(np.float64)
    return cfg, X, C, v, dev(X), dev(C), dev(v)


def test_fullsize_one_sided_and_fused(ctx, full_problem):
    cfg, X, C, v, dX, dC, dv = full_problem
    rng = np.random.default_rng(cfg.seed)
    rows = np.sort(rng.choice(cfg.n, 48, replace=False))
    cols = np.sort(rng.choice(cfg.m, 8, replace=False))
    # pass A on sampled rows
    w = host(ctx.kernel_vec(dX, dC, dv, G, cfg.sigma, zeros(cfg.n)))
    w_ref = oracle.knm_vec(X[rows], C, v, G, cfg.sigma)
    assert rel_l2(w[rows], w_ref) <= TOL
    # pass B on sampled centers, driven by the GPU's full w
    u1 = host(ctx.kernel_tvec(dX, dC, dev(w), G, cfg.sigma, zeros(cfg.m)))
    u1_ref = oracle.knm_t_vec(X, C[cols], w, G, cfg.sigma)
    assert rel_l2(u1[cols], u1_ref) <= TOL
    # the fused product equals the composition (it rounds w to fp32 internally)
    u = host(ctx.knm_matvec(dX, dC, dv, G, cfg.sigma, zeros(cfg.m)))
    assert rel_l2(u, u1) <= TOL


def test_fullsize_sigma_infinity(ctx, full_problem):
    cfg, X, C, v, dX, dC, dv = full_problem
    va = np.abs(v)
    u = host(ctx.knm_matvec(dX, dC, dev(va), G, 1e6, zeros(cfg.m)))
    assert np.max(np.abs(u - cfg.n * va.sum())) <= 1e-6 * cfg.n * va.sum()
