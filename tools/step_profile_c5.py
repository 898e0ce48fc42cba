"""Per-step update-launch times of one C5 factorization (n = 131,072, tile
512), for A/B comparisons between builds.  Prints one JSON line."""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.getcwd()
sys.path.insert(0, ROOT)
from paper_1305_4886_b200 import distla, spawn  # noqa: E402

n, b = 131072, 512
X = np.random.default_rng(0).uniform(0, 1, (n, 2))
cl = spawn(1, tile=b)
lay = distla.make_layout(n, cl.grid)
cl.push("in", {"coords": X})
out = []
for rep in range(2):
    C = distla.construct_distributed(cl, "C", "triangular", "gen.sqexp-nugget.cov", [1.0, 0.02, 0.1],
                                     inputs_name="in", row_layout=lay)
    cl.lib.bgp_set_profiling(cl._ctx, 1)
    prof = (ctypes.c_double * 10)()
    cl.lib.bgp_profile_read(cl._ctx, prof)
    cl.synchronize()
    t = time.perf_counter()
    distla.distributed_cholesky(cl, C, "L")
    wall = time.perf_counter() - t
    cl.lib.bgp_profile_read(cl._ctx, prof)
    steps = (ctypes.c_double * 4096)()
    ns = cl.lib.bgp_profile_steps(cl._ctx, steps, 4096)
    cl.lib.bgp_set_profiling(cl._ctx, 0)
    cl.remote_rm("L")
    out.append({"wall_s": wall, "factor_ms": prof[8], "gemm_ms": prof[2], "steps_ms": [round(steps[i], 4) for i in range(ns)]})
print(json.dumps(out[-1]))
cl.shutdown()
