"""Diagnostic: GSC-Falkon (Alg. 2) GPU vs oracle per Newton step, per
product path and contraction precision, plus the CONDITIONING of the oracle's own answer: its
alpha after each step when every coordinate of X and C is perturbed by one fp32 ulp-level
relative noise (6e-8), i.e. by less than the GPU's own rounding of the kernel values.
    python scripts/gsc_diag.py n m d sigma  (e.g. 4097 257 90 7.0)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle import gsc_oracle as gsc
from paper_2006_10350_b200 import binding

n, m, d, sigma = [float(x) if i == 3 else int(x) for i, x in enumerate(sys.argv[1:5])]
X = synth.gen_X(3, 0, n, d); y = synth.gen_y(3, X, 0, "cls")
idx = synth.center_indices(3, n, m); C, yC = X[idx].copy(), y[idx].copy()
mus, its = [1e-3, 1e-4, 1e-5, 1e-6], [4, 4, 4, 8]
ctx = binding.Context(0)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
out = {"n": n, "m": m, "d": d, "sigma": sigma}
ref = {k: gsc.gsc_falkon(X, y, C, yC, gsc.LOGISTIC, 0, sigma, mus[:k], its[:k]) for k in range(1, 5)}
rng = np.random.default_rng(5)
Xp = (X.astype(np.float64) * (1 + 6e-8 * rng.standard_normal(X.shape))).astype(np.float32)
Cp = Xp[idx].copy()
for k in range(1, 5):
    out[f"oracle_noise6e-8_steps{k}"] = rel(gsc.gsc_falkon(Xp, y, Cp, yC, gsc.LOGISTIC, 0, sigma, mus[:k], its[:k]), ref[k])
for path in (0, 1):
    for acc in (0, 1):
        ctx.set_option(binding.OPT_PATH, path)
        ctx.set_option(binding.OPT_ACCUM_F64, acc)
        for k in range(1, 5):
            a = torch.zeros(m, dtype=torch.float64, device="cuda")
            ctx.gsc_fit(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(C).cuda(),
                        torch.from_numpy(yC).cuda(), 0, sigma, "logistic", mus[:k], its[:k], a)
            out[f"gpu_path{path}_f64{acc}_steps{k}"] = rel(a.cpu().numpy(), ref[k])
print(json.dumps(out))
