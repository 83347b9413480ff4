"""SIMT / tensor crossover on d at large n (FALKON_OPT_TC_MIN_D): one Gaussian product per path
at n = 1e7, m = 2e4 for d = 4..10 (the n-sweep shows n-independent rates beyond n ~ 3e5)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = [sys.argv[0], "none"]
import mvm_sweep as ms  # noqa: E402
from paper_2006_10350_b200 import binding  # noqa: E402
ctx = binding.Context(0)
for d in (4, 5, 6, 7, 8, 9, 10):
    for path in ("simt", "tensor"):
        print(json.dumps({"sweep": "crossover", **ms.measure(ctx, 10_000_000, 20_000, d, 1.5, binding.GAUSSIAN, path, reps=3)}), flush=True)
