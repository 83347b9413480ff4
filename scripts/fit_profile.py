"""Time one falkon_fit with per-class kernel timing (prep/passA/passB/precond/trsv/vec)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2006_10350_b200 import binding

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="msd"); ap.add_argument("--n", type=int); ap.add_argument("--m", type=int)
ap.add_argument("--iters", type=int); ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
n = a.n or cfg.n; m = a.m or cfg.m
X = synth.gen_X(cfg.seed, 0, n, cfg.d)
y = synth.gen_y(cfg.seed, X, 0, cfg.task)
C = synth.gen_rows(cfg.seed, synth.STREAM_X, synth.center_indices(cfg.seed, n, m), cfg.d)
ctx = binding.Context(0)
dX, dy, dC = (torch.from_numpy(t).cuda() for t in (X, y, C))
alpha = torch.zeros(m, dtype=torch.float64, device="cuda")
for r in range(a.repeat):
    ctx.set_option(binding.OPT_KERNEL_TIMING, 1)
    ctx.timings(reset=True)
    t0 = time.perf_counter()
    _, info = ctx.fit(dX, dy, dC, 0, cfg.sigma, cfg.lam, a.iters or cfg.iters, alpha)
    wall = time.perf_counter() - t0
    print(json.dumps({"config": a.config, "n": n, "m": m, "wall_s": wall, "info": info,
                      "kernel_ms": ctx.timings()}), flush=True)
