"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): tcgen05 two-pass (resident d = 90, clusters on and off), streaming
d = 440 + single evaluation (k strip + GEMV), fp64 contractions, SIMT small-d and generic,
multi-vector, the fp64 preconditioner (DMMA GEMMs incl. the TMA-fed variant, diagonal blocks,
distributed schedule) and the sentinel TRSV, one small fit."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synth
from paper_2006_10350_b200 import binding

ctx = binding.Context(0)
G, L = binding.GAUSSIAN, binding.LAPLACIAN
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
z = lambda n: torch.zeros(n, dtype=torch.float64, device="cuda")
for (n, m, d, s) in [(700, 300, 90, 7.0), (520, 300, 440, 14.5), (900, 200, 9, 1.0), (300, 100, 40, 3.0)]:
    X = synth.gen_X(1, 0, n, d); C = X[:m].copy(); v = np.ones(m)
    for opt in ((binding.OPT_TC_CLUSTER, 1), (binding.OPT_TC_CLUSTER, 2)):
        ctx.set_option(*opt)
        ctx.knm_matvec(dev(X), dev(C), dev(v), G, s, z(m))
    ctx.set_option(binding.OPT_ACCUM_F64, 1)
    ctx.knm_matvec(dev(X), dev(C), dev(v), G, s, z(m))
    ctx.set_option(binding.OPT_ACCUM_F64, 0)
    ctx.knm_matvec(dev(X), dev(C), dev(v), L, s, z(m))
    ctx.set_option(binding.OPT_SINGLE_EVAL, 1); ctx.set_option(binding.OPT_STRIP_BYTES, 64 << 20)
    ctx.knm_matvec(dev(X), dev(C), dev(v), G, s, z(m))
    ctx.set_option(binding.OPT_SINGLE_EVAL, 2)
    V = np.ones((m, 16)); ctx.knm_matmat(dev(X), dev(C), dev(V), G, s, z(m * 16).reshape(m, 16))
cfg, X, y, C = synth.make_problem("msd", n=3000, m=600)
ctx.set_option(binding.OPT_POTRF_OUTER, 1)
a, info = ctx.fit(dev(X), dev(y), dev(C), G, cfg.sigma, cfg.lam, 3, z(600))
P = torch.zeros((600, 600), dtype=torch.float64, device="cuda")
bufs = [(torch.zeros((600, 600), dtype=torch.float64, device="cuda"), z(600), z(600),
         z(ctx.precond_work_elems(600))) for _ in range(2)]
ctx.precond_build_sim(dev(C), G, cfg.sigma, cfg.lam, 1e-8, *[list(x) for x in zip(*bufs)])
torch.cuda.synchronize()
print("sanitize cases done")
