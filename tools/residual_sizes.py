"""Large factorizations (step pairs at tile 512, the 256 / 128 tail levels,
the multi-step tail) checked by residual probes ||L L^T x - C x|| / ||C x||
computed on the device (bgp_tri_mv), for sizes too large for a host LAPACK
check.  One JSON line per size.

    python tools/residual_sizes.py [n1,n2,...] [tile]     (GPU)
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_4886_b200 import distla, spawn  # noqa: E402


def p(t):
    return ctypes.c_void_p(t.data_ptr())


def main():
    sizes = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "33100,40000,52001").split(",")]
    tile = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    cl = spawn(1, tile=tile)
    for n in sizes:
        X = np.random.default_rng(n).uniform(0, 1, (n, 2))
        lay = distla.make_layout(n, cl.grid)
        cl.push("in", {"coords": X, "nu": 0.5})
        theta = [1.0, 0.08, 0.02]
        distla.construct_distributed(cl, "C", "triangular", "gen.matern-nugget.cov", theta, inputs_name="in",
                                     row_layout=lay)
        L, _ = distla.distributed_cholesky(cl, distla.DistTriangular("C", lay), "L")
        distla.construct_distributed(cl, "C2", "triangular", "gen.matern-nugget.cov", theta, inputs_name="in",
                                     row_layout=lay)
        Lo, Co = cl.fetch("L"), cl.fetch("C2")
        probes = []
        for seed in range(2):
            x = np.random.default_rng(seed).standard_normal(n)
            xd = cl.fetch(distla.distribute(cl, "x", x, "vector", lay).name).data
            t1, t2, cx = torch.zeros_like(xd), torch.zeros_like(xd), torch.zeros_like(xd)
            cl.call("bgp_tri_mv", p(Lo.data), n, tile, p(xd), p(t1), 1, cl.stream)
            cl.call("bgp_tri_mv", p(Lo.data), n, tile, p(t1), p(t2), 0, cl.stream)
            cl.call("bgp_tri_mv", p(Co.data), n, tile, p(xd), p(cx), 2, cl.stream)
            probes.append(float(torch.linalg.norm((t2 - cx)[:n]) / torch.linalg.norm(cx[:n])))
        print(json.dumps({"n": n, "tile": tile, "T": -(-n // tile), "residual_probes": probes}), flush=True)
        for k in ("L", "C2", "x"):
            cl.remote_rm(k)
    cl.shutdown()


if __name__ == "__main__":
    main()
