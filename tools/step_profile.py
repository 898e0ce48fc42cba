"""Per-step efficiency of the C4 factorization (look-ahead schedule).

    python tools/step_profile.py [--tile 512] > gpurun_out/steps.json
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1305_4886_b200 import spawn  # noqa: E402
from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tile", type=int, default=512)
args = ap.parse_args()
d = np.load(os.path.join(ROOT, "tests", "golden", "c4_inputs.npz"))
X, y = d["X"], d["y"]
cl = spawn(1, tile=args.tile)
prob = KrigeProblem(cl, "p", builtin_spec("matern-nugget", X, nu=0.5), y, [1.0, 0.08, 0.02])
prob.log_density(np.array([1.0, 0.08, 0.02]))
lib, ctx = cl.lib, cl._ctx
lib.bgp_set_profiling(ctx, 1)
prob.log_density(np.array([1.0, 0.08 + 1e-12, 0.02]))
buf = (ctypes.c_double * 4096)()
nst = lib.bgp_profile_steps(ctx, buf, 4096) + 1  # + the re-tiled tail, if any
b = args.tile
T = (len(y) + b - 1) // b
out = []
for J in range(nst):
    k = T - J - 1
    fl = b ** 3 * (k * k + max(k - 1, 0))
    out.append({"J": J, "k": k, "ms": buf[J], "tflops": fl / (buf[J] * 1e-3) / 1e12 if buf[J] > 0 else 0})
print(json.dumps(out))
cl.shutdown()
