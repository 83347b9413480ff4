"""Config-scale fit parity (north_star: alpha and predictions within 1e-3 of
the fp64 oracle).  The oracle fits are stored in tests/golden/fits/*.npz, written by
scripts/oracle_golden.py (which calls only oracle/ and synth/; oracle wall times of hours on a
host CPU, hence stored).  Each golden names its config, n (full or a row prefix) and m; the GPU
fit runs on the same seeded inputs through the C ABI with the library's default precision and
is compared on alpha and on 10,000 held-out predictions.
"""
import glob
import json
import os

import numpy as np
import pytest

import synth
from gpu_util import dev, host, rel_l2, zeros

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "fits", "*.npz")))


@pytest.mark.parametrize("accum_f64", [0, 1], ids=["default", "accum_f64"])
@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[:-4] for p in GOLD])
def test_fit_matches_stored_oracle(ctx, path, accum_f64):
    from paper_2006_10350_b200 import binding
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    cfg = synth.CONFIGS[meta["config"]]
    _, X, y, C = synth.make_problem(meta["config"], n=meta["n"], m=meta["m"])
    Xs = synth.gen_X(cfg.seed, 0, meta["n_test"], cfg.d, stream=synth.STREAM_XTEST)
    ctx.set_option(binding.OPT_ACCUM_F64, accum_f64)
    try:
        alpha, info = ctx.fit(dev(X), dev(y), dev(C), meta["kernel"], meta["sigma"], meta["lam"],
                              meta["iters"], zeros(meta["m"]), meta["jitter"])
    finally:
        ctx.set_option(binding.OPT_ACCUM_F64, 0)
    assert info["iters_run"] == meta["iters_run"]
    f = host(ctx.predict(dev(Xs), dev(C), alpha, meta["kernel"], meta["sigma"],
                         zeros(meta["n_test"])))
    ea, ef = rel_l2(host(alpha), z["alpha"]), rel_l2(f, z["pred"])
    print(json.dumps({"golden": os.path.basename(path), "accum_f64": accum_f64,
                      "alpha_rel_l2": float(ea), "pred_rel_l2": float(ef),
                      "product_path": info.get("product_path")}))
    assert ea <= 1e-3, f"alpha rel-L2 {ea:.2e}"
    assert ef <= 1e-3, f"prediction rel-L2 {ef:.2e}"
