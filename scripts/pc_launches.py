"""One precond_build at m (env PC_M, default 50000) after a tiny warm-up: run under
`ncu --metrics gpu__time_duration.sum` to get the per-kernel split of the preconditioner."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2006_10350_b200 import binding

ctx = binding.Context(0)
cfg = synth.CONFIGS["msd"]
ms = [int(os.environ.get("PC_M", "50000"))]
if os.environ.get("PC_WARM", "1") == "1":
    ms = [1000] + ms
for m in ms:
    C = torch.randn(m, cfg.d, dtype=torch.float32, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(m))
    P = torch.empty(m * m, dtype=torch.float64, device="cuda")
    dT = torch.empty(m, dtype=torch.float64, device="cuda")
    dA = torch.empty(m, dtype=torch.float64, device="cuda")
    W = torch.empty(binding.Context.precond_work_elems(m), dtype=torch.float64, device="cuda")
    ctx.precond_build(C, 0, cfg.sigma, cfg.lam, 1e-8, P, dT, dA, W)
    torch.cuda.synchronize()
    del P
