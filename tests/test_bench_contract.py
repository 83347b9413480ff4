"""The bench.py contract on CPU (-m "not gpu"): the reference arm (the CPU oracle, tier
framing) prints ONE JSON line with the driver's keys, rank > 0 prints nothing, and the roofline
helper's algorithmic work matches SURVEY.md §8(d)'s per-entry figures."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=300, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_reference_arm_json_line():
    lines = _run(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1",
                  "--oracle-seconds", "0.5"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["unit"] == "n*m/s" and d["config"]["workload"] == "tiny"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_nonzero_rank_is_silent():
    lines = _run(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "1",
                  "--oracle-seconds", "0.2"], env={"RANK": "1", "WORLD_SIZE": "2"})
    assert lines == []


def test_roofline_algorithmic_work():
    """tensor path: achieved TFLOP/s = 2 d n m / t; SIMT: evals / t against min(FP32, MUFU)."""
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    import synth
    args = argparse.Namespace(path="auto", steps=1, single_eval=None)
    cfg = synth.CONFIGS["msd"]
    kt = {"pass_a": (10.0, 1), "pass_b": (9.0, 1)}
    r = bench.roofline(args, cfg, kt, 20.0, cfg.n, cfg.m, 148)
    assert r["bound"] == "tensor" and r["kernel"] == "pass_a"
    assert abs(r["achieved"] - 2 * cfg.d * cfg.n * cfg.m / 10e-3 / 1e12) < 1e-9
    cfg = synth.CONFIGS["tiny"]
    r = bench.roofline(args, cfg, kt, 20.0, cfg.n, cfg.m, 148)
    assert r["bound"] == "alu" and r["unit"] == "G kernel-evals/s"
    assert abs(r["achieved"] - cfg.n * cfg.m / 10e-3 / 1e9) < 1e-9


def test_roofline_single_evaluation_strips():
    """TIMIT (d = 440) takes the single-evaluation product by default: pass A runs once per row
    strip, so the per-launch work is n m / launches; the strip GEMV gets an HBM roofline at
    4 B per entry."""
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    import synth
    cfg = synth.CONFIGS["timit"]
    args = argparse.Namespace(path="auto", steps=2, single_eval=None)
    assert bench.single_eval_active(args, cfg.d)
    kt = {"pass_a": (520.0, 52), "pass_b": (140.0, 52)}  # 26 strips x 2 products
    r = bench.roofline(args, cfg, kt, 700.0, cfg.n, cfg.m, 148)
    assert r["kernel"] == "pass_a" and r["launches"] == 52
    assert abs(r["achieved"] - 2 * cfg.d * cfg.n * cfg.m * 2 / 520e-3 / 1e12) < 1e-6
    g = r["strip_gemv"]
    assert g["bound"] == "hbm" and abs(g["achieved"] - 4 * cfg.n * cfg.m * 2 / 140e-3 / 1e9) < 1e-6
    assert not bench.single_eval_active(argparse.Namespace(path="auto", single_eval=None),
                                        synth.CONFIGS["msd"].d)


def test_gpus_flag_spawns_ranks_reference_arm():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself as 2 ranks
    (torch.distributed.run on 127.0.0.1); the reference arm then prints exactly ONE line
    (rank 0) reporting n_gpus = 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--config", "tiny", "--steps", "1", "--warmup", "1",
                        "--oracle-seconds", "0.2"], capture_output=True, text=True, timeout=300,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_product_roofline_fraction_i():
    """frac_product (SURVEY.md §8(d) fraction (i)): the single-evaluation roofline is the
    tensor fp32-class rate / 2d for MSD/TIMIT, the MUFU ex2 rate for HIGGS/TAXI (tensor cross
    term not binding) and min(FP32/(d+3), MUFU) on the SIMT path."""
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    import synth
    peaks, _ = bench.measured_peaks()
    f = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    a = argparse.Namespace(path="auto")
    pk, _ = bench.product_roofline(a, synth.CONFIGS["timit"], 148)
    assert abs(pk - float(peaks["bf16_tflops"]) / 3 * 1e12 / 880) < 1.0
    pk, _ = bench.product_roofline(a, synth.CONFIGS["higgs"], 148)
    assert abs(pk - 148 * 16 * f) < 1.0
    pk, _ = bench.product_roofline(argparse.Namespace(path="simt"), synth.CONFIGS["taxi"], 148)
    assert abs(pk - min(148 * 128 * f / 12, 148 * 16 * f)) < 1.0
