"""Diagnostic: relative error statistics of the kernel values K(x_i, c_j) the GPU paths use,
against fp64 (oracle.kernel_block), on config-shaped synthetic data.  Row i of K is read as
Knm^T e_i through falkon_kernel_tvec (fp64 accumulation so the only error is k's own)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, synth
from paper_2006_10350_b200 import binding

ctx = binding.Context(0)
ctx.set_option(binding.OPT_ACCUM_F64, 1)
for name in sys.argv[1:] or ["taxi", "higgs", "msd", "timit"]:
    cfg = synth.CONFIGS[name]
    n, m = 4000, 3000
    _, X, y, C = synth.make_problem(name, n=n, m=m)
    Xd, Cd = torch.from_numpy(X).cuda(), torch.from_numpy(C).cuda()
    rows = list(range(0, 64))
    Kref = oracle.kernel_block(X[rows], C, oracle.GAUSSIAN, cfg.sigma)
    for path, pid in (("tensor", binding.PATH_TENSOR), ("simt", binding.PATH_SIMT)):
        ctx.set_option(binding.OPT_PATH, pid)
        K = np.zeros_like(Kref)
        for t, i in enumerate(rows):
            e = torch.zeros(n, dtype=torch.float64, device="cuda")
            e[i] = 1.0
            u = torch.zeros(m, dtype=torch.float64, device="cuda")
            ctx.kernel_tvec(Xd, Cd, e, oracle.GAUSSIAN, cfg.sigma, u)
            K[t] = u.cpu().numpy()
        mask = Kref > 1e-6
        r = (K[mask] / Kref[mask] - 1.0)
        t_ref = np.log2(Kref[mask])
        # error of the exponent t = log2 K, per row: mean (systematic per row) and spread
        dt = np.log2(K[mask] / Kref[mask])
        print(json.dumps({"config": name, "path": path, "entries": int(mask.sum()),
                          "rel_mean": float(r.mean()), "rel_std": float(r.std()),
                          "rel_absmax": float(np.abs(r).max()),
                          "dt_std": float(dt.std()), "dt_mean": float(dt.mean()),
                          "t_abs_mean": float(np.abs(t_ref).mean())}), flush=True)
    ctx.set_option(binding.OPT_PATH, binding.PATH_AUTO)
