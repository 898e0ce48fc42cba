"""One warm-up + one profiled C4 log-likelihood evaluation (for ncu captures).

    python tools/profile_c4.py [--tile 256] [--evals 1]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1305_4886_b200 import spawn  # noqa: E402
from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tile", type=int, default=512)
ap.add_argument("--evals", type=int, default=1)
ap.add_argument("--n", type=int, default=0)
args = ap.parse_args()
d = np.load(os.path.join(ROOT, "tests", "golden", "c4_inputs.npz"))
X, y = d["X"], d["y"]
if args.n:
    X, y = X[:args.n], y[:args.n]
cl = spawn(1, tile=args.tile)
prob = KrigeProblem(cl, "p", builtin_spec("matern-nugget", X, nu=0.5), y, [1.0, 0.08, 0.02])
for k in range(1 + args.evals):
    t = time.perf_counter()
    ll = prob.log_density(np.array([1.0, 0.08 + k * 1e-12, 0.02]))
    print(f"eval {k}: ll={ll:.10f} {time.perf_counter() - t:.3f} s", flush=True)
cl.shutdown()
