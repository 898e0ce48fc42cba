"""Per-step efficiency of the factorization (look-ahead schedule) and the
phase split of one log_density, for C4 (frozen inputs) or C2 (seeded recipe).

    python tools/step_profile.py [--config 4] [--tile 512] > gpurun_out/steps.json
"""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1305_4886_b200 import spawn  # noqa: E402
from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tile", type=int, default=512)
ap.add_argument("--config", type=int, default=4)
args = ap.parse_args()
cl = spawn(1, tile=args.tile)
if args.config == 4:
    d = np.load(os.path.join(ROOT, "tests", "golden", "c4_inputs.npz"))
    X, y = d["X"], d["y"]
    spec, theta = builtin_spec("matern-nugget", X, nu=0.5), np.array([1.0, 0.08, 0.02])
else:
    from oracle.blockgp_oracle import config_inputs
    kern, X, theta, extra, z = config_inputs(args.config)
    spec = builtin_spec(kern, X, **extra)
    y = np.random.default_rng(0).standard_normal(len(X))  # timing only
prob = KrigeProblem(cl, "p", spec, y, theta)
prob.log_density(theta)
lib, ctx = cl.lib, cl._ctx
lib.bgp_set_profiling(ctx, 1)
prof = (ctypes.c_double * 10)()
lib.bgp_profile_read(ctx, prof)
th = theta.copy()
th[1] += 1e-12
torch.cuda.synchronize()
t0 = time.perf_counter()
prob.log_density(th)
torch.cuda.synchronize()
eval_ms = 1e3 * (time.perf_counter() - t0)
lib.bgp_profile_read(ctx, prof)
buf = (ctypes.c_double * 4096)()
nst = lib.bgp_profile_steps(ctx, buf, 4096) + 1  # + the re-tiled tail, if any
b = args.tile
T = (len(y) + b - 1) // b
steps = []
for J in range(nst):
    k = T - J - 1
    fl = b ** 3 * (k * k + max(k - 1, 0))
    steps.append({"J": J, "k": k, "ms": buf[J], "tflops": fl / (buf[J] * 1e-3) / 1e12 if buf[J] > 0 else 0})
n = len(y)
print(json.dumps({"config": args.config, "n": n, "tile": b, "eval_ms_wall": eval_ms,
                  "cholesky_ms": prof[8], "potrf_ms": prof[0], "potrf_exposed_ms": prof[9],
                  "trsm_ms": prof[1], "gemm_ms": prof[2], "gemm_launches": prof[3],
                  "cholesky_tflops": n ** 3 / 3 / (prof[8] * 1e-3) / 1e12 if prof[8] else None,
                  "steps": steps}))
cl.shutdown()
