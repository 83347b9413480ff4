"""Diagnostic: GSC (Alg. 2) GPU vs oracle error per Newton step and per product path."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from oracle import gsc
from paper_2006_10350_b200 import binding

n, m, d, sigma = [float(x) if i == 3 else int(x) for i, x in enumerate(sys.argv[1:5])]
X = synth.gen_X(3, 0, n, d); y = synth.gen_y(3, X, 0, "cls")
idx = synth.center_indices(3, n, m); C, yC = X[idx].copy(), y[idx].copy()
mus, its = [1e-3, 1e-4, 1e-5, 1e-6], [4, 4, 4, 8]
ctx = binding.Context(0)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
out = {}
for path in (0, 1):
    ctx.set_option(binding.OPT_PATH, path)
    for k in range(1, 5):
        a = torch.zeros(m, dtype=torch.float64, device="cuda")
        ctx.gsc_fit(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(C).cuda(),
                    torch.from_numpy(yC).cuda(), 0, sigma, "logistic", mus[:k], its[:k], a)
        ao = gsc.gsc_falkon(X, y, C, yC, gsc.LOGISTIC, 0, sigma, mus[:k], its[:k])
        out[f"path{path}_steps{k}"] = rel(a.cpu().numpy(), ao)
    for lam in (1e-3, 1e-5, 1e-6):
        a = torch.zeros(m, dtype=torch.float64, device="cuda")
        ctx.fit(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), torch.from_numpy(C).cuda(), 0, sigma, lam, 8, a)
        out[f"path{path}_falkon_lam{lam}"] = rel(a.cpu().numpy(), oracle.fit(X, y, C, 0, sigma, lam, 8))
    # single product accuracy
    v = np.random.default_rng(0).standard_normal(m)
    u = torch.zeros(m, dtype=torch.float64, device="cuda")
    ctx.knm_matvec(torch.from_numpy(X).cuda(), torch.from_numpy(C).cuda(), torch.from_numpy(v).cuda(), 0, sigma, u)
    out[f"path{path}_product"] = rel(u.cpu().numpy(), oracle.knm_t_knm_vec(X, C, v, 0, sigma))
print(json.dumps(out))
