"""Product throughput sweeps mirroring the paper's Fig. `mvm_impl` (SURVEY.md
§8(d)): n-sweep at m = 2e4, d = 10 and d-sweep at m = n = 2e4, both product paths (SIMT FP32
and tcgen05 tensor), plus Laplacian-kernel lines at the HIGGS and TAXI shapes (SIMT only,
direct differences, reading c7) against their FP32/MUFU roofline.

One JSON line per point: n*m/s of one fused Knm^T(Knm v) (CUDA events over `reps` products,
inputs resident), and the single-evaluation roofline fraction of the path.

    python scripts/mvm_sweep.py [n|d|lap|all]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2006_10350_b200 import binding  # noqa: E402

SMS = 148
F_HZ = 1965e6
PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1671.0}


def roofline(path, kernel, d):
    mufu = SMS * 16 * F_HZ
    if kernel == binding.LAPLACIAN:  # 2d + 3 FP32 ops + 2 MUFU (rsqrt/sqrt, ex2) per entry
        return min(SMS * 128 * F_HZ / (2 * d + 3), mufu / 2)
    if path == "tensor":
        return min(float(PEAKS["bf16_tflops"]) / 3 * 1e12 / (2 * d), mufu)
    return min(SMS * 128 * F_HZ / (d + 3), mufu)


def measure(ctx, n, m, d, sigma, kernel, path, reps=None, seed=7):
    X = synth.gen_X_torch(seed, 0, n, d)
    C = synth.gen_X_torch(seed + 1, 0, m, d)
    v = torch.randn(m, dtype=torch.float64, device="cuda")
    u = torch.zeros(m, dtype=torch.float64, device="cuda")
    ctx.set_option(binding.OPT_PATH, {"simt": binding.PATH_SIMT, "tensor": binding.PATH_TENSOR}[path])
    for _ in range(2):
        ctx.knm_matvec(X, C, v, kernel, sigma, u)
    torch.cuda.synchronize()
    if reps is None:  # ~0.3 s of work
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.knm_matvec(X, C, v, kernel, sigma, u)
        e1.record()
        torch.cuda.synchronize()
        reps = int(max(3, min(200, 300.0 / max(e0.elapsed_time(e1), 1e-3))))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ctx.knm_matvec(X, C, v, kernel, sigma, u)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rate = n * m / (ms * 1e-3)
    rf = roofline(path, kernel, d)
    return {"n": n, "m": m, "d": d, "kernel": "laplacian" if kernel else "gaussian", "path": path,
            "ms": ms, "nm_per_s": rate, "roofline_nm_per_s": rf, "frac_product": rate / rf,
            "reps": reps}


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    ctx = binding.Context(0)
    G, L = binding.GAUSSIAN, binding.LAPLACIAN
    if what in ("n", "all"):
        for n in (100_000, 300_000, 1_000_000, 3_000_000, 10_000_000, 30_000_000, 100_000_000):
            for path in ("simt", "tensor"):
                print(json.dumps({"sweep": "n", **measure(ctx, n, 20_000, 10, 3.0, G, path)}),
                      flush=True)
    if what in ("d", "all"):
        for d in (2, 3, 4, 6, 8, 9, 10, 12, 16, 20, 28, 32, 48, 64, 90, 128, 190, 256, 440, 512,
                  1024):
            for path in ("simt", "tensor"):
                if path == "simt" and d > 256:
                    continue  # the generic SIMT kernel at d > 256: minutes per point, not a contender
                print(json.dumps({"sweep": "d", **measure(ctx, 20_000, 20_000, d,
                                                          max(1.0, np.sqrt(d) / 2), G, path)}),
                      flush=True)
    if what in ("lap", "all"):
        for name, n in (("higgs", 1_000_000), ("taxi", 10_000_000)):
            cfg = synth.CONFIGS[name]
            r = measure(ctx, n, cfg.m, cfg.d, cfg.sigma, L, "simt", reps=3)
            print(json.dumps({"sweep": "laplacian", "shape": name, **r}), flush=True)
            r = measure(ctx, n, cfg.m, cfg.d, cfg.sigma, G, "simt", reps=3)
            print(json.dumps({"sweep": "gaussian_simt", "shape": name, **r}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
