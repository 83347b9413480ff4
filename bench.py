#!/usr/bin/env python
"""Benchmark of the Falkon hot path on B200 (contract: see DESIGN.md "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config msd] [--impl ours|reference]

One STEP = one fused product  u = sum_ranks Knm_r^T (Knm_r v)  (SURVEY.md §8(a) rows a1-a6:
prep, cross term, exp, both contractions, deterministic reduction, allreduce) over the
config's synthetic data, inputs resident in HBM.  metric = n*m kernel evaluations per second
(whole job, all ranks).  After the timed product steps one full falkon_fit (rows a1-a9, the
paper's Table 1 split) is timed and reported under "fit".

Multi-GPU: launched by torch.distributed.run; rows of X are sharded (synth.shard_range), C
and v are replicated, one NCCL allreduce(m) per product; timing is max over ranks.
`--impl reference` times the CPU oracle (oracle/, fp64 NumPy) on a bounded row sample of
the same workload on rank 0 (the only other place allowed to execute oracle/).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


L2_BYTES = 126 << 20  # B200 L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="timit", choices=list(synth.CONFIGS),
                    help="BASELINE.json workload (default: TIMIT, the largest single-GPU config)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-fit", action="store_true", help="skip the full falkon_fit timing")
    ap.add_argument("--fit-iters", type=int, default=None)
    ap.add_argument("--path", default="auto", choices=["auto", "simt", "tensor", "f64"])
    ap.add_argument("--n", type=int, default=None, help="override global n (debug)")
    ap.add_argument("--m", type=int, default=None, help="override m (debug)")
    ap.add_argument("--oracle-seconds", type=float, default=15.0)
    ap.add_argument("--exp-offload", type=int, default=None,
                    help="tensor path: exp2 share on the FMA pipe (0 none, 1 all, 2 1/4, 3 1/2)")
    ap.add_argument("--gsc-config", default=None, choices=[None] + list(synth.GSC_CONFIGS),
                    help="also time one GSC-Falkon / LogFalkon fit (Alg. 2) on this workload")
    ap.add_argument("--gsc-n", type=int, default=None, help="override the GSC workload's n")
    ap.add_argument("--single-eval", type=int, default=None, choices=[0, 1, 2],
                    help="products: 0 two passes, 1 single evaluation (k strip), 2 auto")
    ap.add_argument("--strip-mb", type=int, default=None,
                    help="single evaluation: k strip budget in MiB (FALKON_OPT_STRIP_BYTES)")
    ap.add_argument("--tc-cluster", type=int, default=None, choices=[1, 2],
                    help="tensor path: 1 CTA or 2-CTA clusters multicasting the Q boxes")
    ap.add_argument("--multi-k", type=int, default=0,
                    help="also time the k-output product Knm^T (Knm V), V in R^{m x k} (NEXT-3)")
    ap.add_argument("--accum-f64", type=int, default=None, choices=[0, 1],
                    help="contractions: 0 fp32 v/w, 1 fp64 v/w with DFMA (FALKON_OPT_ACCUM_F64)")
    ap.add_argument("--quick", action="store_true",
                    help="timed product steps only (no e2e, cpu_baseline, fit): for ncu runs")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a torchrun environment: re-launch this script as N
    ranks (one process per GPU) through torch.distributed.run on 127.0.0.1.  Rank 0 prints the
    JSON line; the return code is torchrun's."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def oracle_rate(cfg, n_global, m, seconds: float, rank_workers: int):
    """Time the fp64 CPU oracle's Knm^T(Knm v) on a bounded row sample of the workload.
    Returns (n*m/s, dict)."""
    import oracle
    C = synth.gen_C(cfg.seed, n_global, m, cfg.d) if m == cfg.m and n_global == cfg.n else \
        synth.gen_rows(cfg.seed, synth.STREAM_X, synth.center_indices(cfg.seed, n_global, m), cfg.d)
    v = synth.gen_vec(cfg.seed, m).astype(np.float64)
    # calibrate on a small sample, then size the sample to ~`seconds`
    q = max(1, (1 << 23) // m)
    n_cal = max(rank_workers * q, 256)
    Xc = synth.gen_X(cfg.seed, 0, n_cal, cfg.d)
    t0 = time.perf_counter()
    oracle.knm_t_knm_vec(Xc, C, v, oracle.GAUSSIAN, cfg.sigma, workers=rank_workers)
    dt = time.perf_counter() - t0
    rate = n_cal * m / dt
    n_s = int(min(n_global, max(n_cal, rate * seconds / m)))
    Xs = synth.gen_X(cfg.seed, 0, n_s, cfg.d)
    t0 = time.perf_counter()
    oracle.knm_t_knm_vec(Xs, C, v, oracle.GAUSSIAN, cfg.sigma, workers=rank_workers)
    dt = time.perf_counter() - t0
    return n_s * m / dt, {"rows": n_s, "m": m, "seconds": dt}


def kt_path_tensor(args, d):
    """Mirror of libfalkon's path choice (tc_supported): tensor cores for the Gaussian kernel
    when d > 4 (measured crossover, profiles/r2_crossover.jsonl), unless --path forces one."""
    if args.path in ("simt", "f64"):
        return False
    return args.path == "tensor" or d > 4


# The paper's whole-fit times on the real datasets (context, not the target).
PAPER_FIT = {
    "msd": "Table 2/4 (PAPER.md:598-601, 846-853): MSD fit 62 s (2x Titan Xp) / 81 s (1x)",
    "timit": "Table 2/4 (PAPER.md:598-601, 846-853): TIMIT fit 288 s (2x Titan Xp) / 416 s (1x)",
    "higgs": "Table 2/4 (PAPER.md:566-569, 846-853): HIGGS fit 443 s (2x Titan Xp) / 715 s (1x)",
    "taxi": "Table 2/4 (PAPER.md:566-569, 846-853): TAXI fit 3628 s (2x Titan Xp) / 7215 s (1x)",
}


def single_eval_active(args, d) -> bool:
    """Mirror of tc_single_eval() in csrc/kvp_tc.cu: single evaluation (k strip) on the tensor
    path when forced, or by default when the padded segment exceeds 192 (d > 190)."""
    if not kt_path_tensor(args, d):
        return False
    se = 2 if args.single_eval is None else args.single_eval
    return se == 1 or (se == 2 and -(-(d + 2) // 16) * 16 > 192)


def roofline(args, cfg, kt, ms_total, n_local, m, sms):
    """Roofline of the dominant kernel (the pass with the larger device time in the timed
    region; both passes evaluate every Knm entry once).  Algorithmic work per launch and
    per entry is SURVEY.md §8(d): the cross term x.c is 2d flops; the exp, bias and
    contraction are 1 exp + 5 flops.

    * tensor path (Gaussian, d > 32): bound "tensor".  The cross term must be fp32-accurate
      (fp16/TF32 single pass fails parity), which tcgen05 delivers as three fp16
      MMAs (fp16x3).  peak = measured bf16/fp16 dense peak / 3 (the fp32-class rate of the
      tensor cores); achieved = 2*d*n*m / kernel time.  `issued_frac` also reports the issued
      fp16 MMA work (3 terms x padded K) against the plain fp16 peak.
    * SIMT path (d <= 32): bound "alu".  Per entry the FP32 pipe executes d FFMA + 1 FADD + 1
      FFMA and the MUFU 1 ex2; peak = min over the two pipes of unit rate x 148 SMs x clock
      (B200: 128 FP32 lanes, 16 MUFU/clk per SM; clock = sm_max_mhz)."""
    peaks, peak_src = measured_peaks()
    dom = max(("pass_a", "pass_b"), key=lambda k: kt[k][0])
    dom_ms = kt[dom][0] / max(1, kt[dom][1])
    # entries per launch of the dominant class: a single-evaluation product launches pass A
    # once per row strip, so the rate is taken over all launches of the timed region
    evals = n_local * m * args.steps * dom_ms / max(kt[dom][0], 1e-9)
    d = cfg.d
    f_hz = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(f"{cfg.name}:{dom}:{n_local}:{m}")
    common = {"kernel": dom, "kernel_ms": dom_ms, "launches": kt[dom][1],
              "share_of_step": kt[dom][0] / ms_total if ms_total else None,
              "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)"}
    if kt_path_tensor(args, d):
        d16 = -(-(d + 2) // 16) * 16  # d coordinates + 2 folded-bias slots (csrc/kvp_tc.cu)
        if d16 > 192:  # streaming kernel: 32-aligned segments
            d16 = -(-(d + 2) // 32) * 32
        peak_tf = float(peaks["bf16_tflops"]) / 3.0
        ach_eval = evals / (dom_ms * 1e-3)
        tc_eval_peak = peak_tf * 1e12 / (2.0 * d)       # fp32-class cross term bound
        mufu_eval_peak = sms * 16 * f_hz               # one ex2 per entry on the MUFU
        issued_tf = 3 * 2.0 * d16 * ach_eval / 1e12
        extra = {"issued_frac": issued_tf / float(peaks["bf16_tflops"]),
                 "evals_per_s": ach_eval, "tensor_evals_peak": tc_eval_peak,
                 "mufu_evals_peak": mufu_eval_peak}
        if single_eval_active(args, d) and kt["pass_b"][1]:
            # second contraction = streaming GEMV over the stored k strip: HBM-bound, 4 B/entry
            gb_s = 4.0 * n_local * m * args.steps / (kt["pass_b"][0] * 1e-3) / 1e9
            extra["single_eval"] = True
            extra["strip_gemv"] = {"bound": "hbm", "achieved": gb_s,
                                   "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                                   "frac": gb_s / float(peaks["hbm_gbs"]),
                                   "ms_per_product": kt["pass_b"][0] / args.steps}
        if tc_eval_peak <= mufu_eval_peak:
            ach_tf = 2.0 * d * ach_eval / 1e12
            sus = peaks.get("bf16_tflops_sustained")
            if sus:  # context only: the power-capped sustained rate (frac uses the burst peak)
                extra["frac_vs_sustained_peak"] = ach_tf / (float(sus) / 3.0)
            return {"bound": "tensor", "achieved": ach_tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": ach_tf / peak_tf,
                    "peak_source": f"{peak_src} bf16 dense {peaks['bf16_tflops']} TF/s / 3 "
                                   "(fp16x3 = fp32-class cross term)", **extra, **common}
        return {"bound": "alu", "pipe": "mufu", "achieved": ach_eval / 1e9,
                "peak": mufu_eval_peak / 1e9, "unit": "G kernel-evals/s",
                "frac": ach_eval / mufu_eval_peak,
                "peak_source": f"{peak_src} sm_max_mhz {f_hz/1e6:.0f} MHz x {sms} SM x 16 MUFU ex2"
                               " per clk (tensor cross term not binding at this d)",
                **extra, **common}
    if args.path == "f64":  # FALKON_PATH_F64: the FP64 pipe (64 DFMA lanes/clk/SM on B200)
        # per entry d cross-term FMAs (DMMA or DFMA: the same fp64 rate on B200) + the fp64 exp2
        # (range reduction + degree-11 polynomial + scaling: 17 operations) + bias + contraction
        peak = sms * 64 * f_hz / (d + 19)
        ach = evals / (dom_ms * 1e-3)
        return {"bound": "alu", "pipe": "fp64", "achieved": ach / 1e9, "peak": peak / 1e9,
                "unit": "G kernel-evals/s", "frac": ach / peak,
                "peak_source": f"sm_max_mhz {f_hz/1e6:.0f} MHz x {sms} SM x 64 fp64 lanes / "
                               "(d + 19) per clk (d cross-term FMAs, 17-op fp64 exp2, bias, "
                               "contraction)", **common}
    fp32 = sms * 128 * f_hz / (d + 2)
    mufu = sms * 16 * f_hz
    peak, pipe = min((fp32, "fp32"), (mufu, "mufu"))
    ach = evals / (dom_ms * 1e-3)
    return {"bound": "alu", "pipe": pipe, "achieved": ach / 1e9, "peak": peak / 1e9,
            "unit": "G kernel-evals/s", "frac": ach / peak,
            "peak_source": f"{peak_src} sm_max_mhz {f_hz/1e6:.0f} MHz x {sms} SM x "
                           "(128 FP32 lanes/(d+2) | 16 MUFU) per clk", **common}


def product_roofline(args, cfg, sms):
    """Single-evaluation roofline of the whole product (SURVEY.md §8(d) fraction (i), the
    headline): per Knm entry the method needs 2d flops of cross term, one bias add, one exp
    and two contraction MACs, evaluated ONCE.  Gaussian: tensor path = min(fp32-class tensor
    rate / 2d, MUFU 16 ex2/clk/SM); SIMT path = min(FP32 128 lanes / (d + 3), MUFU).
    Returns (kernel evals/s per GPU, description)."""
    peaks, src = measured_peaks()
    f_hz = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    d = cfg.d
    mufu = sms * 16 * f_hz
    if kt_path_tensor(args, d):
        tc = float(peaks["bf16_tflops"]) / 3.0 * 1e12 / (2.0 * d)
        pk = min(tc, mufu)
        return pk, (f"min(tensor {peaks['bf16_tflops']} TF/s / 3 / 2d = {tc:.3g}, MUFU "
                    f"{sms} SM x 16 x {f_hz/1e6:.0f} MHz = {mufu:.3g}) evals/s ({src} peaks)")
    if args.path == "f64":
        pk = sms * 64 * f_hz / (d + 19)
        return pk, f"FP64 {sms} SM x 64 lanes x {f_hz/1e6:.0f} MHz / (d + 19) evals/s"
    fp32 = sms * 128 * f_hz / (d + 3)
    pk = min(fp32, mufu)
    return pk, (f"min(FP32 {sms} SM x 128 x {f_hz/1e6:.0f} MHz / (d+3) = {fp32:.3g}, MUFU "
                f"{mufu:.3g}) evals/s")


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    n_global = args.n or cfg.n
    m = args.m or cfg.m
    cores = host_cores()
    steps_v = []
    info = None
    per_step = max(2.0, min(args.oracle_seconds, 60.0 / max(1, args.steps + args.warmup)))
    for i in range(args.warmup + args.steps):
        v, info = oracle_rate(cfg, n_global, m, per_step, cores)
        if i >= args.warmup:
            steps_v.append((v, info))
    vals = [s[0] for s in steps_v]
    value = statistics.median(vals)
    ms = float(np.median([s[1]["seconds"] for s in steps_v])) * 1e3
    out = {
        "impl": "reference", "metric": "fused Knm^T(Knm v) kernel-evals/s", "value": value,
        "unit": "n*m/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (synth/, seeded; shapes of BASELINE.json configs)",
        "config": {"workload": cfg.name, "n": n_global, "d": cfg.d, "m": m, "sigma": cfg.sigma,
                   "kernel": "gaussian"},
        "cpu_baseline": {"value": value, "unit": "n*m/s", "cores": cores, "kind": "oracle",
                         "sample": f"{info['rows']} of {n_global} rows x all {m} centers per step "
                                   f"(fp64 NumPy oracle, {cores} worker processes)"},
        "e2e": {"value": value, "unit": "n*m/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_gsc(args, ctx, world, rank, barrier):
    """One GSC-Falkon / LogFalkon fit (Alg. 2) on this rank's shard of
    a GSC workload (synth.GSC_CONFIGS), timed host call -> return (max over ranks)."""
    import torch
    import torch.distributed as dist
    g = synth.GSC_CONFIGS[args.gsc_config]
    base = synth.CONFIGS[g.base]
    n_global = args.gsc_n or base.n
    lo, hi = synth.shard_range(n_global, world, rank)
    X = synth.gen_X(base.seed, lo, hi - lo, base.d)
    y = synth.gen_y(base.seed, X, lo, "cls")
    idx = synth.center_indices(base.seed, n_global, g.m)
    C = synth.gen_rows(base.seed, synth.STREAM_X, idx, base.d)
    yC = synth.gen_y_rows(base.seed, C, idx, "cls")
    Xd, yd, Cd, yCd = (torch.from_numpy(a).cuda() for a in (X, y, C, yC))
    alpha = torch.zeros(g.m, dtype=torch.float64, device="cuda")
    try:
        barrier()
        t0 = time.perf_counter()
        _, info = ctx.gsc_fit(Xd, yd, Cd, yCd, "gaussian", g.sigma, "logistic", list(g.mus),
                              list(g.iters), alpha)
        barrier()
        wall = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([wall], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall = float(t.item())
        return {"workload": g.name, "n": n_global, "d": base.d, "m": g.m, "sigma": g.sigma,
                "newton_steps": len(g.mus), "cg_iters": int(sum(g.iters)), "seconds": wall,
                "t_precond_s": info["t_precond_s"], "t_rhs_s": info["t_rhs_s"],
                "t_cg_s": info["t_cg_s"], "iters_run": info["iters_run"],
                "paper_context": "Table 2 (PAPER.md:571-573): LogFalkon HIGGS 2267 s "
                                 "(2x Titan Xp, full HIGGS)"}
    except Exception as ex:  # report, do not hide
        return {"workload": g.name, "error": str(ex)}


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world, rank, local = dist_env()
    if args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; timing {world} ranks",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2006_10350_b200 import binding

    from paper_2006_10350_b200 import parallel

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    ctx = parallel.make_context(local, world, rank, stream=stream)
    ctx.set_option(binding.OPT_PATH, {"auto": 0, "simt": 1, "tensor": 2, "f64": 3}[args.path])
    if args.exp_offload is not None:
        ctx.set_option(binding.OPT_EXP_OFFLOAD, args.exp_offload)
    if args.single_eval is not None:
        ctx.set_option(binding.OPT_SINGLE_EVAL, args.single_eval)
    if args.strip_mb is not None:
        ctx.set_option(binding.OPT_STRIP_BYTES, args.strip_mb << 20)
    if args.accum_f64 is not None:
        ctx.set_option(binding.OPT_ACCUM_F64, args.accum_f64)
    if args.tc_cluster is not None:
        ctx.set_option(binding.OPT_TC_CLUSTER, args.tc_cluster)

    n_global = args.n or cfg.n
    m = args.m or cfg.m
    lo, hi = synth.shard_range(n_global, world, rank)
    n_local = hi - lo
    # ---- inputs (seeded, synthetic; generated on the host and uploaded once, or generated
    # on the device with the same hash when too large for the host, e.g. TAXI 1e9 x 9) ----
    big = n_local * cfg.d > 600_000_000
    Ch = torch.from_numpy(synth.gen_rows(cfg.seed, synth.STREAM_X,
                                         synth.center_indices(cfg.seed, n_global, m), cfg.d)
                          ).pin_memory()
    vh = torch.from_numpy(synth.gen_vec(cfg.seed, m).astype(np.float64)).pin_memory()
    if big:
        Xh = None
        X = synth.gen_X_torch(cfg.seed, lo, n_local, cfg.d, device="cuda")
        args.no_fit = args.no_fit or args.fit_iters is None
    else:
        Xh = torch.from_numpy(synth.gen_X(cfg.seed, lo, n_local, cfg.d)).pin_memory()
        X = Xh.cuda()
    C, v = Ch.cuda(), vh.cuda()
    u = torch.zeros(m, dtype=torch.float64, device="cuda")
    kernel, sigma = binding.GAUSSIAN, cfg.sigma

    def step():
        ctx.knm_matvec(X, C, v, kernel, sigma, u)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    ctx.set_option(binding.OPT_KERNEL_TIMING, 1)
    ctx.timings(reset=True)
    l0 = ctx.launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    # Inputs smaller than 2x L2 (e.g. a rank's shard at N > 1) get an L2 flush between the
    # timed steps (a 512 MB write, outside the per-step events); larger inputs stream anyway.
    packed = n_local * (2 * 2 * (-(-(cfg.d + 2) // 16) * 16) if kt_path_tensor(args, cfg.d)
                        else 4 * (-(-cfg.d // 4) * 4))
    flush = packed < 2 * L2_BYTES
    fbuf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if flush else None
    barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps if flush else 1)]
    if flush:
        for i in range(args.steps):
            fbuf.fill_(i & 0xFF)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
    else:
        evs[0][0].record(stream)
        for _ in range(args.steps):
            step()
        evs[0][1].record(stream)
    barrier()
    clk = clocks.stop()
    ms_total = sum(a.elapsed_time(b) for a, b in evs)
    kt = ctx.timings(reset=True)
    launches = ctx.launch_count() - l0 - kt["allreduce"][1]
    ctx.set_option(binding.OPT_KERNEL_TIMING, 0)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = n_global * m / (ms_step * 1e-3)

    # ---- roofline of the dominant kernel (device-timed inside the timed region) ----
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    roof = roofline(args, cfg, kt, ms_total, n_local, m, sms)
    pk_evals, pk_desc = product_roofline(args, cfg, sms)
    roof["frac_product"] = value / world / pk_evals  # fraction (i): whole product, per GPU
    roof["product_roofline"] = {"evals_per_s": pk_evals, "basis": pk_desc}

    if args.quick:
        args.no_fit = True
    # ---- e2e: same metric through the C-ABI with HOST (pinned) buffers ----
    uh = torch.zeros(m, dtype=torch.float64).pin_memory()
    e2e_steps = 0 if (args.quick or Xh is None) else max(3, min(args.steps, 10))
    for _ in range(2 if e2e_steps else 0):
        ctx.knm_matvec(Xh, Ch, vh, kernel, sigma, uh)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ctx.knm_matvec(Xh, Ch, vh, kernel, sigma, uh)
    barrier()
    e2e_s = (time.perf_counter() - t0) / max(1, e2e_steps)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = None if not e2e_steps else {"value": n_global * m / e2e_s, "unit": "n*m/s",
           "h2d_bytes_per_step": int(Xh.numel() * 4 + Ch.numel() * 4 + vh.numel() * 8),
           "d2h_bytes_per_step": int(uh.numel() * 8)}

    # ---- one full Falkon fit (rows a1-a9) ----
    fit = None
    if not args.no_fit:
        if Xh is None:  # device-generated X (TAXI-size): targets generated on the device too
            y = synth.gen_y_torch(cfg.seed, X, lo, cfg.task)
        else:
            y = torch.from_numpy(synth.gen_y(cfg.seed, Xh.numpy(), lo, cfg.task)).cuda()
        alpha = torch.zeros(m, dtype=torch.float64, device="cuda")
        iters = args.fit_iters if args.fit_iters is not None else cfg.iters
        try:
            barrier()
            t0 = time.perf_counter()
            _, info = ctx.fit(X, y, C, kernel, sigma, cfg.lam, iters, alpha)
            barrier()
            wall = time.perf_counter() - t0
            fit = {"seconds": wall, "iters": iters, "t_precond_s": info["t_precond_s"],
                   "t_rhs_s": info["t_rhs_s"], "t_cg_s": info["t_cg_s"],
                   "iters_run": info["iters_run"],
                   # product kernels the fit ran on (readings d3 / d4)
                   "product_path": {1: "simt", 2: "tensor", 3: "f64"}.get(info.get("product_path"),
                                                                           info.get("product_path")),
                   "paper_context": PAPER_FIT.get(cfg.name)}
        except Exception as ex:  # report, do not hide
            fit = {"error": str(ex)}

    multi = None
    if args.multi_k > 0:
        k = args.multi_k
        V = torch.from_numpy(np.random.default_rng(7).standard_normal((m, k))).cuda()
        U = torch.zeros((m, k), dtype=torch.float64, device="cuda")
        for _ in range(2):
            ctx.knm_matmat(X, C, V, kernel, sigma, U)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(2, min(args.steps, 5))
        e0.record(stream)
        for _ in range(reps):
            ctx.knm_matmat(X, C, V, kernel, sigma, U)
        e1.record(stream)
        barrier()
        ms_k = e0.elapsed_time(e1) / reps
        if world > 1:
            t = torch.tensor([ms_k], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_k = float(t.item())
        multi = {"k": k, "ms_per_product": ms_k, "value": n_global * m * k / (ms_k * 1e-3),
                 "unit": "n*m*k/s", "vs_k_single_products": k * ms_step / ms_k}

    gsc_fit = None
    if args.gsc_config and not args.quick:
        gsc_fit = run_gsc(args, ctx, world, rank, barrier)

    cpu = None
    if rank == 0 and world == 1 and not args.quick:
        rate, inf = oracle_rate(cfg, n_global, m, args.oracle_seconds, host_cores())
        cpu = {"value": rate, "unit": "n*m/s", "cores": host_cores(), "kind": "oracle",
               "sample": f"{inf['rows']} of {n_global} rows x all {m} centers, one product, "
                         f"{inf['seconds']:.1f} s (fp64 NumPy oracle, {host_cores()} worker procs)"}

    if rank == 0:
        out = {
            "metric": "fused Knm^T(Knm v) kernel-evals/s", "value": value, "unit": "n*m/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (synth/, seeded; "
            "X ~ N(0,1) fp32, C = uniform rows of X; shapes of BASELINE.json)",
            "config": {"workload": cfg.name, "n": n_global, "d": cfg.d, "m": m,
                       "sigma": cfg.sigma, "kernel": "gaussian",
                       "path": "tensor" if kt_path_tensor(args, cfg.d) else "simt",
                       "parallelism": f"rows sharded dp{world}, allreduce(m) per product",
                       "l2": ("L2 flushed between timed steps (512 MB write, untimed; packed X "
                              "%.0f MB < 2x L2)" if flush else "inputs larger than L2 (packed X "
                              "%.0f MB)") % (packed / 1e6)},
            "clocks": clk, "gpu_launches": int(launches), "roofline": roof, "e2e": e2e,
            "cpu_baseline": cpu, "fit": fit, "gsc_fit": gsc_fit, "multi_output": multi,
            "kernel_ms": {k: v[0] for k, v in kt.items()},
        }
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
