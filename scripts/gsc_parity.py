"""GSC-Falkon / LogFalkon parity at a larger HIGGS-shaped prefix: GPU falkon_gsc_fit vs the
oracle's Alg. 2 on the same seeded inputs (alpha and held-out prediction rel. L2)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from oracle import gsc
from paper_2006_10350_b200 import binding

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="higgs_log")
ap.add_argument("--n", type=int, default=200_000)
ap.add_argument("--m", type=int, default=2_000)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
g, X, y, C, yC = synth.make_gsc_problem(a.config, n=a.n, m=a.m)
mus = list(np.geomspace(1e-3, 1e-9, a.steps)) if a.steps > 1 else [1e-9]
its = [5] * (a.steps - 1) + [10]
base = synth.CONFIGS[g.base]
Xs = synth.gen_X(base.seed, 0, 4000, base.d, stream=synth.STREAM_XTEST)
ctx = binding.Context(0)
alpha = torch.zeros(a.m, dtype=torch.float64, device="cuda")
t0 = time.time()
_, info = ctx.gsc_fit(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(C).cuda(),
                      torch.from_numpy(yC).cuda(), 0, g.sigma, "logistic", mus, its, alpha)
torch.cuda.synchronize(); t_gpu = time.time() - t0
f = torch.zeros(4000, dtype=torch.float64, device="cuda")
ctx.predict(torch.from_numpy(Xs).cuda(), torch.from_numpy(C).cuda(), alpha, 0, g.sigma, f)
alpha, f = alpha.cpu().numpy(), f.cpu().numpy()
t0 = time.time()
aref = gsc.gsc_falkon(X, y, C, yC, gsc.LOGISTIC, 0, g.sigma, mus, its)
t_cpu = time.time() - t0
fref = oracle.predict(Xs, C, aref, 0, g.sigma)
rel = lambda u, v: float(np.linalg.norm(u - v) / np.linalg.norm(v))
print(json.dumps({"config": a.config, "n": a.n, "m": a.m, "d": base.d, "sigma": g.sigma,
                  "mus": mus, "iters": its, "alpha_rel_l2": rel(alpha, aref),
                  "pred_rel_l2": rel(f, fref), "sign_agreement": float(np.mean(np.sign(f) == np.sign(fref))),
                  "gpu_fit_s": t_gpu, "oracle_fit_s": t_cpu, "gpu_info": info}), flush=True)
