"""FALKON_TC_PAIR A/B: CTA-pair (cta_group::2) streaming kernel vs oracle, several shapes."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, synth
from paper_2006_10350_b200 import binding
ctx = binding.Context(0)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for (n, m, d, s, se, acc) in [(3000, 700, 440, 14.5, 0, 0), (3000, 700, 440, 14.5, 1, 0), (2999, 513, 300, 12.0, 1, 1),
                              (4001, 900, 256, 10.0, 0, 1), (700, 300, 440, 14.5, 2, 0)]:
    X = synth.gen_X(d, 0, n, d); C = X[synth.center_indices(d, n, m)]; v = synth.gen_vec(d, m).astype(np.float64)
    ctx.set_option(binding.OPT_SINGLE_EVAL, se); ctx.set_option(binding.OPT_ACCUM_F64, acc)
    u = torch.zeros(m, dtype=torch.float64, device="cuda")
    ctx.knm_matvec(dev(X), dev(C), dev(v), 0, s, u)
    ref = oracle.knm_t_knm_vec(X, C, v, 0, s)
    print(n, m, d, se, acc, "rel", float(np.linalg.norm(u.cpu().numpy() - ref) / np.linalg.norm(ref)), flush=True)
