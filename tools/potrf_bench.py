"""Device time of the tile POTRF and of POTRF + inverse (one CTA each), per
tile size: the serial link of every factorization step.

    python tools/potrf_bench.py
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_4886_b200 import spawn  # noqa: E402

reps = 50
for b in (128, 256, 512):
    cl = spawn(1, tile=b)
    B = np.random.default_rng(0).standard_normal((b, b))
    A = B @ B.T + b * np.eye(b)
    t0 = torch.from_numpy(np.tril(A).T.copy()).to(cl.device)
    works = [torch.empty_like(t0) for _ in range(reps)]
    linv = torch.empty_like(t0)
    s = cl.stream
    out = {"tile": b}
    for name, inv in (("potrf_us", None), ("potrf_inv_us", linv)):
        for w in works:
            w.copy_(t0)
        cl.lib.bgp_info_reset(cl._ctx, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for w in works:
            cl.lib.bgp_tile_potrf_async(cl._ctx, ctypes.c_void_p(w.data_ptr()), b, 0,
                                        ctypes.c_void_p(inv.data_ptr()) if inv is not None else None, s)
        e1.record()
        torch.cuda.synchronize()
        out[name] = round(e0.elapsed_time(e1) / reps * 1e3, 1)
    L = np.tril(works[-1].cpu().numpy().T)
    out["err"] = float(np.abs(L @ L.T - A).max() / np.abs(A).max())
    print(json.dumps(out), flush=True)
    cl.shutdown()
