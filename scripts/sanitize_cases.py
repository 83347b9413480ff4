"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): tcgen05 two-pass (resident d = 90, clusters on and off), streaming
d = 440 + single evaluation (k strip + GEMV), fp64 contractions, SIMT small-d and generic,
multi-vector, the fp64 preconditioner (DMMA GEMMs incl. the TMA-fed variant, diagonal blocks,
distributed schedule, the Ozaki int8 GEMMs incl. the LAUUM chunks) and the sentinel TRSV, the
fp64 product path (DMMA / DFMA / chunked kernels), the split-SM strip GEMV, one small fit."""
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
# Ozaki GEMMs (m >= 512; the potrf_outer = 1 above keeps k = 128 panels on DMMA, so reset it)
ctx.set_option(binding.OPT_POTRF_OUTER, 8)
Cz = synth.gen_X(2, 0, 1300, 28)
Pz = torch.zeros((1300, 1300), dtype=torch.float64, device="cuda")
ctx.precond_build(dev(Cz), G, 3.8, 1e-6, 1e-8, Pz, z(1300), z(1300), z(ctx.precond_work_elems(1300)))
# fp64 product path: DMMA (Gaussian d <= 64), DFMA (Laplacian), chunked (d > 64)
ctx.set_option(binding.OPT_PATH, binding.PATH_F64)
for (n, m, d, kern) in [(700, 300, 28, G), (700, 300, 28, L), (300, 150, 90, G)]:
    X = synth.gen_X(3, 0, n, d); C = X[:m].copy(); v = np.ones(m)
    ctx.knm_matvec(dev(X), dev(C), dev(v), kern, 4.0, z(m))
ctx.set_option(binding.OPT_PATH, binding.PATH_AUTO)
# split-SM strip GEMV (second stream)
X = synth.gen_X(4, 0, 9000, 300); C = X[:500].copy(); v = np.ones(500)
ctx.set_option(binding.OPT_SINGLE_EVAL, 1); ctx.set_option(binding.OPT_STRIP_BYTES, 64 << 20)
ctx.set_option(binding.OPT_SE_GEMV_SMS, 8)
ctx.knm_matvec(dev(X), dev(C), dev(v), G, 12.0, z(500))
ctx.set_option(binding.OPT_SE_GEMV_SMS, 0); ctx.set_option(binding.OPT_SINGLE_EVAL, 2)
torch.cuda.synchronize()
print("sanitize cases done")
