"""GPU tests of the distributed preconditioner (App. C
Alg. 3/4): the 1D block-cyclic schedule (panel j owned by rank j mod G, owner factors, panel
broadcast, every rank updates its own column panels, LAUUM split by column panels).

* G ranks simulated in one process (falkon_precond_build_sim): every rank's factors are
  BITWISE equal to the single-GPU build with the same blocking, and match the oracle.
* the real NCCL path on one GPU (1-rank communicator, FALKON_OPT_DIST_PRECOND): bitwise equal,
  and a full fit through it.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = pytest.mark.gpu
G = oracle.GAUSSIAN


def _bufs(ctx, m):
    import torch
    P = torch.full((m, m), float("nan"), dtype=torch.float64, device="cuda")
    return P, zeros(m), zeros(m), zeros(ctx.precond_work_elems(m))


def _factors(P, dT, dA):
    Ph = host(P)
    T = np.triu(Ph, 1) + np.diag(host(dT))
    A = (np.tril(Ph, -1) + np.diag(host(dA))).T
    return T, A


def _parts(P, dT, dA, W):
    Ph = host(P)
    return np.triu(Ph, 1), np.tril(Ph, -1), host(dT), host(dA), host(W)


@pytest.fixture()
def ctx1(lib):
    """A fresh context per test (the options below change the blocking)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2006_10350_b200 import binding
    c = binding.Context(device=0)
    yield c
    c.close()


@pytest.mark.parametrize("Gr", [1, 2, 3, 8])
@pytest.mark.parametrize("m,d,outer", [(700, 9, 1), (1300, 28, 2), (2600, 90, 8)])
def test_simulated_ranks_bitwise_equal_single_gpu(ctx1, Gr, m, d, outer):
    from paper_2006_10350_b200 import binding
    ctx1.set_option(binding.OPT_POTRF_OUTER, outer)  # outer panels of outer x 128 columns
    X = synth.gen_X(50 + d, 0, 4 * m, d)
    C = X[synth.center_indices(50 + d, 4 * m, m)]
    sigma, lam = 2.0, 1e-6
    ref = _bufs(ctx1, m)
    ctx1.precond_build(dev(C), G, sigma, lam, 1e-8, *ref)
    bufs = [_bufs(ctx1, m) for _ in range(Gr)]
    ctx1.precond_build_sim(dev(C), G, sigma, lam, 1e-8, [b[0] for b in bufs], [b[1] for b in bufs],
                           [b[2] for b in bufs], [b[3] for b in bufs])
    want = _parts(*ref)
    for r in range(Gr):
        got = _parts(*bufs[r])
        for a, b in zip(got, want):
            assert np.array_equal(a, b), f"rank {r} differs from the single-GPU build"
    # and the oracle (fp64 on both sides)
    T, A = _factors(*bufs[-1][:3])
    To, Ao = oracle.preconditioner(C, G, sigma, lam, 1e-8)
    assert rel_l2(T, To) <= 1e-9 and rel_l2(A, Ao) <= 1e-9


def test_simulated_ranks_report_not_pd(ctx1):
    """A pivot failure in one owner's panel reaches every rank (ENOTPD, same column as the
    single-GPU build)."""
    from paper_2006_10350_b200 import binding
    ctx1.set_option(binding.OPT_POTRF_OUTER, 1)
    X = synth.gen_X(61, 0, 600, 5)
    C = np.concatenate([X[:300], X[:300]])  # duplicated centres, no jitter: Kmm singular
    ref = _bufs(ctx1, 600)
    with pytest.raises(binding.FalkonError) as e1:
        ctx1.precond_build(dev(C), G, 1.0, 1e-6, 0.0, *ref)
    bufs = [_bufs(ctx1, 600) for _ in range(3)]
    with pytest.raises(binding.FalkonError) as e2:
        ctx1.precond_build_sim(dev(C), G, 1.0, 1e-6, 0.0, [b[0] for b in bufs],
                               [b[1] for b in bufs], [b[2] for b in bufs], [b[3] for b in bufs])
    assert e1.value.code == e2.value.code == 2
    assert e1.value.info["failed_column"] == e2.value.info["failed_column"]


def test_nccl_path_one_rank_bitwise_and_fit(lib):
    """The real distributed path (NCCL broadcasts on the context's communicator) on a 1-rank
    communicator: same bits as the single-GPU build, and falkon_fit through it matches."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2006_10350_b200 import binding
    uid = binding.get_unique_id()
    c = binding.Context(device=0, rank=0, world=1, unique_id=uid)
    c0 = binding.Context(device=0)
    try:
        for cc in (c, c0):
            cc.set_option(binding.OPT_POTRF_OUTER, 1)
        c.set_option(binding.OPT_DIST_PRECOND, 1)
        cfg, X, y, C = synth.make_problem("msd", n=6000, m=900)
        a, b = _bufs(c, 900), _bufs(c0, 900)
        c.precond_build(dev(C), G, cfg.sigma, cfg.lam, 1e-8, *a)
        c0.precond_build(dev(C), G, cfg.sigma, cfg.lam, 1e-8, *b)
        for x, y_ in zip(_parts(*a), _parts(*b)):
            assert np.array_equal(x, y_)
        al, _ = c.fit(dev(X), dev(y), dev(C), G, cfg.sigma, cfg.lam, cfg.iters, zeros(900))
        a0, _ = c0.fit(dev(X), dev(y), dev(C), G, cfg.sigma, cfg.lam, cfg.iters, zeros(900))
        assert np.array_equal(host(al), host(a0))
    finally:
        c.close()
        c0.close()
