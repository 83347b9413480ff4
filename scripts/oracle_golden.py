"""Write oracle fits to tests/golden/fits/ for the config-scale GPU parity tests.

Calls ONLY oracle/ (and synth/ for the seeded inputs): the stored alpha and held-out
predictions are the fp64 CPU oracle's (Alg. 1), never the CUDA path's.

    python scripts/oracle_golden.py --config msd                 # full n, config m
    python scripts/oracle_golden.py --config higgs --n 1050000 --m 50000

Output: tests/golden/fits/<config>_n<n>_m<m>[_lap].npz with alpha (m fp64), pred (10,000
held-out rows of the XTEST stream, fp64) and a JSON `meta` string (shape, hyper-parameters,
oracle wall time, host cores).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

N_TEST = 10_000


def golden_path(config: str, n: int, m: int, kernel: int = 0) -> str:
    lap = "_lap" if kernel == oracle.LAPLACIAN else ""
    return os.path.join(ROOT, "tests", "golden", "fits", f"{config}_n{n}_m{m}{lap}.npz")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--n", type=int)
    ap.add_argument("--m", type=int)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--direct-max-d", type=int, default=None,
                    help="oracle: direct differences only up to this d (default: the oracle's "
                         "DIRECT_DIFF_MAX_D = 32); above it the fp64 norm expansion (error ~1e-13 "
                         "relative on the squared distance, SURVEY.md E4), ~10x faster at d = 28")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    n, m = a.n or cfg.n, a.m or cfg.m
    out = golden_path(a.config, n, m, a.kernel)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if a.direct_max_d is not None:
        from oracle import falkon_oracle as fo
        fo.DIRECT_DIFF_MAX_D = a.direct_max_d  # forked product workers inherit it
    t0 = time.time()
    _, X, y, C = synth.make_problem(a.config, n=n, m=m)
    Xs = synth.gen_X(cfg.seed, 0, N_TEST, cfg.d, stream=synth.STREAM_XTEST)
    t1 = time.time()
    alpha, info = oracle.fit(X, y, C, a.kernel, cfg.sigma, cfg.lam, cfg.iters,
                             workers=a.workers, return_info=True)
    t2 = time.time()
    pred = oracle.predict(Xs, C, alpha, a.kernel, cfg.sigma)
    meta = {"config": a.config, "n": n, "m": m, "d": cfg.d, "sigma": cfg.sigma, "lam": cfg.lam,
            "iters": cfg.iters, "kernel": a.kernel, "jitter": oracle.DEFAULT_JITTER,
            "iters_run": info["iters_run"], "n_test": N_TEST, "test_stream": synth.STREAM_XTEST,
            "oracle_fit_s": round(t2 - t1, 1), "gen_s": round(t1 - t0, 1),
            "workers": a.workers, "host_cores": os.cpu_count(),
            "direct_diff_max_d": a.direct_max_d if a.direct_max_d is not None else 32,
            "writer": "scripts/oracle_golden.py (oracle/ only)"}
    del info
    np.savez(out, alpha=alpha, pred=pred, meta=json.dumps(meta))
    print(json.dumps({"out": os.path.relpath(out, ROOT), **meta}), flush=True)


if __name__ == "__main__":
    main()
