"""Per-launch timeline of the look-ahead chain (probe build with
-DBGP_EXP_LTRACE, tools: see DESIGN 9).  Runs one C2-size log_density.
    BGP_LIB_PATH=build/probe/libbgp_LT.so python tools/ltrace_c2.py [tile]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.blockgp_oracle import config_inputs  # noqa: E402
from paper_1305_4886_b200 import spawn  # noqa: E402
from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec  # noqa: E402

tile = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cl = spawn(1, tile=tile)
kern, X, theta, extra, z = config_inputs(2)
prob = KrigeProblem(cl, "p", builtin_spec(kern, X, **extra), np.random.default_rng(0).standard_normal(len(X)), theta)
prob.log_density(theta)
lib = cl.lib
lib.bgp_probe_ltrace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((8192, 8), dtype=np.uint64)
torch.cuda.synchronize()
lib.bgp_probe_ltrace(None, 1)
th = np.array(theta, dtype=float)
th[1] += 1e-12
prob.log_density(th)
torch.cuda.synchronize()
lib.bgp_probe_ltrace(ctypes.c_void_p(buf.ctypes.data), 0)
rows = [r for r in buf.astype(np.int64) if r[7] > 0 and r[6] > 0]
print("launches", len(rows))
prev_end = None
for r in rows:
    t0 = r[0]
    f = lambda k: (r[k] - t0) / 1e3 if r[k] > 0 and r[k] != -1 else float("nan")  # noqa: E731
    gap = (t0 - prev_end) / 1e3 if prev_end else float("nan")
    print(f"T={r[7]:3d} gap_us={gap:7.1f} diag_gate={f(1):7.1f} potrf_inv_done={f(2):7.1f} "
          f"trsm_first={f(3):7.1f} trsm_last={f(4):7.1f} upd_last={f(5):7.1f} exit={f(6):7.1f}")
    prev_end = r[6]
cl.shutdown()
