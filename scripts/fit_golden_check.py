"""GPU fits vs the stored oracle fits of tests/golden/fits/ (written by scripts/oracle_golden.py,
oracle-only): alpha and held-out prediction relative L2 for each precision / path variant.
One JSON line per (golden, variant).  Usage: python scripts/fit_golden_check.py [glob]"""
import glob, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synth
from paper_2006_10350_b200 import binding

pat = sys.argv[1] if len(sys.argv) > 1 else "*"
# (name, fp64 contractions, path (0 auto, 1 SIMT, 3 fp64), exp on the FMA pipe, Ozaki, FIT_PRECISE)
variants = [("default", 0, 0, 0, 1, 1), ("fp32_noprecise", 0, 0, 0, 1, 0),
            ("f64contr_noprecise", 1, 0, 0, 1, 0), ("simt_fp32", 0, 1, 0, 1, 0),
            ("f64path", 0, 3, 0, 1, 1), ("dmma_precond", 0, 0, 0, 0, 1)]
if len(sys.argv) > 2:
    variants = [v for v in variants if v[0] in sys.argv[2].split(",")]
ctx = binding.Context(0)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for f in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "fits", pat + ".npz"))):
    z = np.load(f)
    meta = json.loads(str(z["meta"]))
    cfg = synth.CONFIGS[meta["config"]]
    _, X, y, C = synth.make_problem(meta["config"], n=meta["n"], m=meta["m"])
    Xs = synth.gen_X(cfg.seed, 0, meta["n_test"], cfg.d, stream=synth.STREAM_XTEST)
    Xd, yd, Cd, Xsd = (torch.from_numpy(a).cuda() for a in (X, y, C, Xs))
    for name, acc, path, expo, oz, precise in variants:
        ctx.set_option(binding.OPT_ACCUM_F64, acc)
        ctx.set_option(binding.OPT_EXP_OFFLOAD, expo)
        ctx.set_option(binding.OPT_OZAKI, oz)
        ctx.set_option(binding.OPT_FIT_PRECISE, precise)
        ctx.set_option(binding.OPT_PATH, path)
        alpha = torch.zeros(meta["m"], dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        t0 = time.time()
        _, info = ctx.fit(Xd, yd, Cd, meta["kernel"], meta["sigma"], meta["lam"], meta["iters"],
                          alpha, meta["jitter"])
        torch.cuda.synchronize()
        t = time.time() - t0
        fp = torch.zeros(meta["n_test"], dtype=torch.float64, device="cuda")
        ctx.predict(Xsd, Cd, alpha, meta["kernel"], meta["sigma"], fp)
        print(json.dumps({"golden": os.path.basename(f), "variant": name, "n": meta["n"],
                          "product_path": info.get("product_path"),
                          "m": meta["m"], "d": cfg.d, "alpha_rel_l2": rel(alpha.cpu().numpy(), z["alpha"]),
                          "pred_rel_l2": rel(fp.cpu().numpy(), z["pred"]), "gpu_fit_s": t,
                          "t_precond_s": info["t_precond_s"], "t_cg_s": info["t_cg_s"],
                          "oracle_fit_s": meta["oracle_fit_s"]}), flush=True)
    ctx.set_option(binding.OPT_PATH, binding.PATH_AUTO)
