"""Probe of the preconditioner's ceilings on the box (diagnostic only, results -> gpurun_out/):
library rates for fp64 GEMM (cuBLAS DGEMM through torch) and int8 GEMM (torch._int_mm) as
context for our DMMA kernel, and the time of libfalkon's precond_build at a few m."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2006_10350_b200 import binding

out = {}
dev = "cuda"


def rate(fn, flops, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e30
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return flops / (best * 1e-3) / 1e12, best


for N in ((4096, 8192) if os.environ.get("PROBE_LIB", "1") == "1" else ()):
    a = torch.randn(N, N, dtype=torch.float64, device=dev)
    b = torch.randn(N, N, dtype=torch.float64, device=dev)
    out[f"cublas_dgemm_{N}_tflops"] = rate(lambda: a @ b, 2.0 * N ** 3)[0]
N = 8192
if os.environ.get("PROBE_LIB", "1") != "1":
    N = 64
a8 = torch.randint(-127, 127, (N, N), dtype=torch.int8, device=dev)
b8 = torch.randint(-127, 127, (N, N), dtype=torch.int8, device=dev).t().contiguous().t()
try:
    out["int8_mm_8192_tops"] = rate(lambda: torch._int_mm(a8, b8), 2.0 * N ** 3)[0]
except Exception as ex:
    out["int8_mm_err"] = str(ex)[:200]
a16 = torch.randn(N, N, dtype=torch.float16, device=dev)
out["fp16_mm_8192_tflops"] = rate(lambda: a16 @ a16, 2.0 * N ** 3)[0]

ctx = binding.Context(0)
import itertools
REF = {}
for la in [int(x) for x in os.environ.get("PROBE_LOOKAHEAD", "1").split(",")]:
 ctx.set_option(binding.OPT_LOOKAHEAD, la)
 for warps, outer in itertools.product([int(x) for x in os.environ.get("PROBE_WARPS", "8").split(",")],
                                      [int(x) for x in os.environ.get("PROBE_OUTER", "8").split(",")]):
  ctx.set_option(binding.OPT_POTRF_OUTER, outer)
  ctx.set_option(binding.OPT_GEMM_WARPS, warps)
  for m in [int(x) for x in os.environ.get("PROBE_M", "20000,50000").split(",")]:
    cfg = synth.CONFIGS["msd"]
    C = torch.randn(m, cfg.d, dtype=torch.float32, device=dev,
                    generator=torch.Generator(device=dev).manual_seed(m))
    P = torch.empty(m * m, dtype=torch.float64, device=dev)
    dT = torch.empty(m, dtype=torch.float64, device=dev)
    dA = torch.empty(m, dtype=torch.float64, device=dev)
    W = torch.empty(binding.Context.precond_work_elems(m), dtype=torch.float64, device=dev)
    ctx.precond_build(C, 0, cfg.sigma, cfg.lam, 1e-8, P, dT, dA, W)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.precond_build(C, 0, cfg.sigma, cfg.lam, 1e-8, P, dT, dA, W)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out[f"precond_la{la}_w{warps}_o{outer}_m{m}_s"] = dt
    key = ("ref", m)
    if key not in REF:
        REF[key] = (P.clone(), dT.clone(), dA.clone())
    else:
        Pr, dTr, dAr = REF[key]
        out[f"precond_la{la}_w{warps}_o{outer}_m{m}_maxdiff"] = max(
            float((P - Pr).abs().max()), float((dT - dTr).abs().max()), float((dA - dAr).abs().max()))
    out[f"precond_la{la}_w{warps}_o{outer}_m{m}_tflops_m3"] = m ** 3 / dt / 1e12
    del P, W
    torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
