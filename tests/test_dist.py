"""Multi-rank (N > 1) host logic of the data-parallel path on CPU: world_size 2 over gloo.

What the GPU path does across ranks: rows sharded with
parallel.shard_range, every m-vector product summed by one allreduce, lambda * n with the
global n, max-over-ranks timing, NCCL id broadcast.  Here the per-rank products come from the
CPU oracle and the allreduce is gloo's, so these tests pin the DECOMPOSITION: the sharded
computation must equal the single-process one.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2006_10350_b200 import parallel

G = oracle.GAUSSIAN


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def test_shard_range_partitions_rows():
    for n in (0, 1, 7, 100, 463715):
        for world in (1, 2, 3, 8):
            spans = [parallel.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
            assert spans == [synth.shard_range(n, world, r) for r in range(world)]


def _sharded_product(rank, world):
    cfg, X, y, C = synth.make_problem("tiny")
    v = synth.gen_vec(cfg.seed, cfg.m).astype(np.float64)
    lo, hi = parallel.shard_range(cfg.n, world, rank)
    u = torch.from_numpy(oracle.knm_t_knm_vec(X[lo:hi], C, v, G, cfg.sigma))
    dist.all_reduce(u)  # the one collective of the product
    return u.numpy()


def test_sharded_product_equals_full_product():
    out = run_world(_sharded_product)
    cfg, X, y, C = synth.make_problem("tiny")
    v = synth.gen_vec(cfg.seed, cfg.m).astype(np.float64)
    full = oracle.knm_t_knm_vec(X, C, v, G, cfg.sigma)
    for r in out:
        assert np.allclose(out[r], full, rtol=1e-12, atol=0)
    assert np.array_equal(out[0], out[1])  # every rank holds identical bits


def _sharded_fit(rank, world):
    """Alg. 1 with row-sharded products and the GLOBAL n in lambda*n (reading c15)."""
    import scipy.linalg as sla
    cfg, X, y, C = synth.make_problem("tiny")
    X, y, C = (a.astype(np.float64) for a in (X, y, C))
    lo, hi = parallel.shard_range(cfg.n, world, rank)
    Xr, yr = X[lo:hi], y[lo:hi]
    n_local = torch.tensor([hi - lo], dtype=torch.int64)
    dist.all_reduce(n_local)
    n_global = int(n_local.item())
    T, A = oracle.preconditioner(C, G, cfg.sigma, cfg.lam)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        return t.numpy()

    c = allreduce(oracle.knm_t_vec(Xr, C, yr, G, cfg.sigma))
    R = sla.solve_triangular(A, sla.solve_triangular(T, c, trans="T"), trans="T")

    def op(beta):
        v = sla.solve_triangular(A, beta)
        cc = allreduce(oracle.knm_t_knm_vec(Xr, C, sla.solve_triangular(T, v), G, cfg.sigma))
        return sla.solve_triangular(A, sla.solve_triangular(T, cc, trans="T")
                                    + cfg.lam * n_global * v, trans="T")

    beta, _ = oracle.conjugate_gradient(op, R, cfg.iters)
    return sla.solve_triangular(T, sla.solve_triangular(A, beta)), n_global


def test_sharded_fit_equals_single_process_fit():
    out = run_world(_sharded_fit)
    cfg, X, y, C = synth.make_problem("tiny")
    ref = oracle.fit(X, y, C, G, cfg.sigma, cfg.lam, cfg.iters)
    for r, (alpha, n_global) in out.items():
        assert n_global == cfg.n
        assert np.linalg.norm(alpha - ref) <= 1e-10 * np.linalg.norm(ref)


def _bootstrap(rank, world):
    uid = parallel.broadcast_bytes(bytes(range(128)) if rank == 0 else None)
    t = parallel.max_over_ranks(float(rank + 1.5))
    return uid, t


def test_unique_id_broadcast_and_max_over_ranks():
    out = run_world(_bootstrap)
    for r, (uid, t) in out.items():
        assert uid == bytes(range(128))
        assert t == 2.5


# ---- NEXT-1: 1D block-cyclic distributed Cholesky (the schedule libfalkon runs across ranks)
def _block_cyclic_cholesky(rank, world, S, nbo):
    """Lower Cholesky S = L L^T with outer panel j owned by rank j % world: the owner factors
    the panel (diagonal block Cholesky + panel solve), broadcasts it, and every rank applies
    the trailing update to ITS column panels only.  Each rank holds a full-size buffer but
    only ever updates its own columns (the storage-replicated layout of csrc/precond.cu)."""
    import scipy.linalg as sla
    m = S.shape[0]
    L = S.copy()
    nob = -(-m // nbo)
    for j in range(nob):
        k0, k1 = j * nbo, min(m, (j + 1) * nbo)
        owner = j % world
        panel = torch.zeros((m - k0, k1 - k0), dtype=torch.float64)
        if rank == owner:
            Lkk = sla.cholesky(L[k0:k1, k0:k1], lower=True)
            L[k0:k1, k0:k1] = Lkk
            if k1 < m:
                L[k1:, k0:k1] = sla.solve_triangular(Lkk, L[k1:, k0:k1].T, lower=True).T
            panel = torch.from_numpy(np.ascontiguousarray(L[k0:, k0:k1]))
        dist.broadcast(panel, src=owner)
        L[k0:, k0:k1] = panel.numpy()
        for c in range(j + 1, nob):
            if c % world != rank:
                continue
            c0, c1 = c * nbo, min(m, (c + 1) * nbo)
            Lp = L[c0:, k0:k1]
            L[c0:, c0:c1] -= Lp @ L[c0:c1, k0:k1].T
    return np.tril(L)


def _dist_precond(rank, world):
    """Both factors of the Falkon preconditioner through the distributed schedule: T^T from
    Kmm + delta I, then A^T from T T^T/m + lam I (LAUUM split by the owners' column panels)."""
    cfg, X, y, C = synth.make_problem("tiny", m=100)
    m, lam, delta = C.shape[0], 1e-3, 1e-8
    K = oracle.kmm(C, G, cfg.sigma) + delta * np.eye(m)
    LT = _block_cyclic_cholesky(rank, world, K, 16)            # L = T^T
    T = LT.T
    M = np.zeros((m, m))
    for c in range(-(-m // 16)):                                  # owned column panels of M
        if c % world == rank:
            c0, c1 = c * 16, min(m, (c + 1) * 16)
            M[:, c0:c1] = (T @ T[c0:c1].T) / m
    Mt = torch.from_numpy(M)
    dist.all_reduce(Mt)  # assemble (each column panel has one writer)
    M = Mt.numpy() + lam * np.eye(m)
    LA = _block_cyclic_cholesky(rank, world, np.tril(M) + np.tril(M, -1).T, 16)
    return T, LA.T


@pytest.mark.parametrize("world", [2, 3])
def test_block_cyclic_preconditioner_decomposition(world):
    out = run_world(_dist_precond, world=world)
    cfg, X, y, C = synth.make_problem("tiny", m=100)
    To, Ao = oracle.preconditioner(C, G, cfg.sigma, 1e-3, 1e-8)
    for r in range(world):
        T, A = out[r]
        assert np.allclose(T, To, rtol=0, atol=1e-12)
        assert np.allclose(A, Ao, rtol=0, atol=1e-10)
        assert np.array_equal(T, out[0][0]) and np.array_equal(A, out[0][1])
