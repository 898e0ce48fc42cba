"""Covariance build (K1) of the C4 triangle at tile 512: median of 7 timed
builds (CUDA events), for A/B of builds via BGP_LIB_PATH.  One JSON line."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1305_4886_b200 import distla, spawn  # noqa: E402

d = np.load(os.path.join(ROOT, "tests", "golden", "c4_inputs.npz"))
X = d["X"]
n = len(X)
cl = spawn(1, tile=512)
lay = distla.make_layout(n, cl.grid)
cl.push("in", {"coords": X, "nu": 0.5})
ts = []
for rep in range(9):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    distla.construct_distributed(cl, "C", "triangular", "gen.matern-nugget.cov", [1.0, 0.08, 0.02],
                                 inputs_name="in", row_layout=lay)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    cl.remote_rm("C")
ts = sorted(ts[2:])
print(json.dumps({"lib": os.environ.get("BGP_LIB_PATH", "default"), "build_ms_median": ts[len(ts) // 2],
                  "min_ms": ts[0], "TBps": 18.104e9 / (ts[len(ts) // 2] * 1e-3) / 1e12}))
cl.shutdown()
