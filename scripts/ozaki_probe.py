"""Preconditioner build time and factor agreement with the Ozaki-scheme trailing updates
(FALKON_OPT_OZAKI = 1) against the fp64 DMMA build, at MSD / TIMIT-class m (one JSON line per m).
    python scripts/ozaki_probe.py [m ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2006_10350_b200 import binding

ctx = binding.Context(0)
if os.environ.get("POTRF_OUTER"):
    ctx.set_option(binding.OPT_POTRF_OUTER, int(os.environ["POTRF_OUTER"]))
for m in [int(x) for x in (sys.argv[1:] or ["20000", "50000"])]:
    cfg = synth.CONFIGS["higgs"]
    C = torch.from_numpy(synth.gen_X(cfg.seed, 0, m, cfg.d)).cuda()
    P = torch.empty(m * m, dtype=torch.float64, device="cuda")
    dT = torch.empty(m, dtype=torch.float64, device="cuda")
    dA = torch.empty(m, dtype=torch.float64, device="cuda")
    W = torch.empty(binding.Context.precond_work_elems(m), dtype=torch.float64, device="cuda")
    rec, ref = {"m": m, "d": cfg.d, "sigma": cfg.sigma}, None
    for oz in (0, 1):
        ctx.set_option(binding.OPT_OZAKI, oz)
        def build():  # FALKON_OZ_DIAG runs produce wrong factors (timing only): ENOTPD ignored
            try:
                ctx.precond_build(C, 0, cfg.sigma, cfg.lam, 1e-8, P, dT, dA, W)
            except binding.FalkonError:
                if not os.environ.get("FALKON_OZ_DIAG"):
                    raise
        build()  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        build()
        torch.cuda.synchronize()
        rec[f"build_s_ozaki{oz}"] = round(time.perf_counter() - t0, 4)
        if os.environ.get("OZ_KERNELS"):  # per-kernel device time (CUPTI through torch.profiler)
            from torch.profiler import profile, ProfilerActivity
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                build()
                torch.cuda.synchronize()
            agg = {}
            for e in prof.events():
                if e.device_type.name == "CUDA":
                    k = e.name.split("(")[0].split("<")[0].replace("void ", "").replace("falkon::", "")
                    agg[k] = agg.get(k, 0.0) + e.device_time_total / 1e3
            rec[f"kernel_ms_ozaki{oz}"] = {k: round(v, 2) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6]}
        if ref is None:
            ref = (P.clone(), dT.clone(), dA.clone())
        else:
            Pu, Pl = torch.triu(P.view(m, m), 1), torch.tril(P.view(m, m), -1)
            Ru, Rl = torch.triu(ref[0].view(m, m), 1), torch.tril(ref[0].view(m, m), -1)
            rec["T_maxdiff_rel"] = float(max((Pu - Ru).abs().max(), (dT - ref[1]).abs().max()) /
                                         max(Ru.abs().max(), ref[1].abs().max()))
            rec["A_maxdiff_rel"] = float(max((Pl - Rl).abs().max(), (dA - ref[2]).abs().max()) /
                                         max(Rl.abs().max(), ref[2].abs().max()))
    ctx.set_option(binding.OPT_OZAKI, 0)
    print(json.dumps(rec), flush=True)
    del P, W
    torch.cuda.empty_cache()
