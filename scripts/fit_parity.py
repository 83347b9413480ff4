"""Fit parity at (near-)config scale: GPU falkon_fit vs the CPU oracle on the same seeded
inputs, reporting alpha and held-out prediction relative L2 errors (north_star bar 1e-3).
Large oracle runs: use on the GPU box's host (many cores); results go to profiles/."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from paper_2006_10350_b200 import binding

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="msd"); ap.add_argument("--n", type=int); ap.add_argument("--m", type=int)
ap.add_argument("--kernel", type=int, default=0)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
n = a.n or cfg.n; m = a.m or cfg.m
cfg2, X, y, C = synth.make_problem(a.config, n=n, m=m)
Xs = synth.gen_X(cfg.seed, 0, 4000, cfg.d, stream=synth.STREAM_XTEST)
ctx = binding.Context(0)
t0 = time.time()
alpha, info = ctx.fit(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(C).cuda(),
                      a.kernel, cfg.sigma, cfg.lam, cfg.iters, torch.zeros(m, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize(); t_gpu = time.time() - t0
f = torch.zeros(4000, dtype=torch.float64, device="cuda")
ctx.predict(torch.from_numpy(Xs).cuda(), torch.from_numpy(C).cuda(), alpha, a.kernel, cfg.sigma, f)
alpha, f = alpha.cpu().numpy(), f.cpu().numpy()
t0 = time.time()
aref = oracle.fit(X, y, C, a.kernel, cfg.sigma, cfg.lam, cfg.iters, workers=len(os.sched_getaffinity(0)))
t_cpu = time.time() - t0
fref = oracle.predict(Xs, C, aref, a.kernel, cfg.sigma)
rel = lambda u, v: float(np.linalg.norm(u - v) / np.linalg.norm(v))
print(json.dumps({"config": a.config, "n": n, "m": m, "d": cfg.d, "sigma": cfg.sigma, "lam": cfg.lam,
                  "iters": cfg.iters, "kernel": a.kernel, "alpha_rel_l2": rel(alpha, aref),
                  "pred_rel_l2": rel(f, fref), "gpu_fit_s": t_gpu, "oracle_fit_s": t_cpu,
                  "gpu_info": info}), flush=True)
