"""Triangular-solve timing on the box (diagnostic): precond at m, then each of the 4 solve
kinds timed with CUDA events (median of 10), with the effective bandwidth over m^2/2 doubles."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2006_10350_b200 import binding

m = int(os.environ.get("TRSV_M", "50000"))
ctx = binding.Context(0)
C = torch.randn(m, 90, dtype=torch.float32, device="cuda")
P = torch.empty(m * m, dtype=torch.float64, device="cuda")
dT = torch.empty(m, dtype=torch.float64, device="cuda")
dA = torch.empty(m, dtype=torch.float64, device="cuda")
W = torch.empty(binding.Context.precond_work_elems(m), dtype=torch.float64, device="cuda")
ctx.precond_build(C, 0, 7.0, 2e-6, 1e-8, P, dT, dA, W)
x0 = torch.randn(m, dtype=torch.float64, device="cuda")
out = {"m": m}
for which in (0, 1):
    for trans in (False, True):
        ts = []
        for _ in range(12):
            x = x0.clone()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); ctx.precond_solve(P, dT, dA, W, which, trans, x); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        med = statistics.median(ts[2:])
        out[f"{'TA'[which]}{'t' if trans else ''}_ms"] = med
        out[f"{'TA'[which]}{'t' if trans else ''}_GBs"] = m * m / 2 * 8 / (med * 1e-3) / 1e9
print(json.dumps(out))
