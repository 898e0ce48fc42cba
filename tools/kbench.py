"""Per-kernel timings at C4-like sizes (CUDA events, after warm-up).

    python tools/kbench.py [--tile 256]

Prints one JSON line per kernel: tile POTRF, panel TRSM (k tiles), a trailing
update step (k tiles), covariance build of T tiles, one TRSV step.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1305_4886_b200 import _lib, spawn  # noqa: E402


def p(t):
    return ctypes.c_void_p(t.data_ptr())


def time_it(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tile", type=int, default=256)
    args = ap.parse_args()
    b = args.tile
    cl = spawn(1, tile=b)
    lib, ctx, s = cl.lib, cl._ctx, cl.stream
    dev = cl.device
    rng = np.random.default_rng(0)
    # an SPD tile (column-major == symmetric)
    B = rng.standard_normal((b, b))
    A = B @ B.T + b * np.eye(b)
    tile0 = torch.from_numpy(np.tril(A).T.copy()).to(dev)
    work = torch.empty_like(tile0)
    info = ctypes.c_int64()

    def potrf():
        work.copy_(tile0)
        lib.bgp_tile_potrf(ctx, p(work), b, 0, ctypes.byref(info), s)

    copy_us = time_it(lambda: work.copy_(tile0))
    us = time_it(potrf) - copy_us
    print(json.dumps({"kernel": "tile_potrf (incl. status sync)", "b": b, "us": round(us, 1),
                      "gflops": round(b ** 3 / 3 / us / 1e3, 1)}))
    linv = torch.empty_like(tile0)

    def potrf_inv():
        work.copy_(tile0)
        lib.bgp_tile_potrf_inv(ctx, p(work), b, p(linv), ctypes.byref(info), s)

    us2 = time_it(potrf_inv) - copy_us
    print(json.dumps({"kernel": "tile_potrf + one-CTA inverse (incl. status sync)", "b": b, "us": round(us2, 1),
                      "inverse_us": round(us2 - us, 1)}))
    L = work.clone()
    for k in (1, 32, 128, 262):
        panel = torch.from_numpy(rng.standard_normal((k, b, b))).to(dev)
        us = time_it(lambda: lib.bgp_panel_trsm(ctx, p(L), p(panel), k, b, s))
        print(json.dumps({"kernel": "panel_trsm", "tiles": k, "us": round(us, 1),
                          "tflops": round(k * b ** 3 / us / 1e6, 2)}))
    # trailing update of one Cholesky step: packed triangle of T tiles, step J
    for T in (32, 96):
        nt = T * (T + 1) // 2
        tiles = torch.from_numpy(rng.standard_normal((nt, b, b)) * 1e-3).to(dev)
        items = []
        k = T - 1
        from paper_1305_4886_b200.parallel import TileDist  # noqa: F401
        def tri(I, J):
            return J * T - J * (J - 1) // 2 + (I - J)
        for C in range(1, T):
            for R in range(C, T):
                items.append((tri(R, C), tri(R, 0), tri(C, 0), int(R == C)))
        it = torch.tensor(np.array(items, dtype=np.int32).ravel(), device=dev)
        us = time_it(lambda: lib.bgp_tile_update(ctx, p(tiles), p(tiles), p(tiles), p(it), len(items), b, s),
                     reps=5)
        flops = b ** 3 * k * k
        print(json.dumps({"kernel": "gemm_dmma (list mode, one step)", "trailing_tiles": k, "us": round(us, 1),
                          "tflops": round(flops / us / 1e6, 2)}))
    # covariance build of 96 x 97 / 2 tiles (exponential)
    n = 96 * b
    X = torch.from_numpy(rng.uniform(0, 1, (n, 2))).to(dev)
    nt = 96 * 97 // 2
    out = torch.empty((nt, b, b), dtype=torch.float64, device=dev)
    g = _lib.Generator(family=_lib.GEN_MATERN, part=_lib.PART_COV, nugget=1, nparams=3, nu=0.5)
    g.params[0], g.params[1], g.params[2] = 1.0, 0.08, 0.02
    us = time_it(lambda: lib.bgp_construct(ctx, _lib.BGP_TRI, ctypes.byref(g), p(X), n, None, 0, 2, b, p(out), s),
                 reps=5)
    gb = 8 * n * (n + 1) / 2 / 1e9
    print(json.dumps({"kernel": "cov_tri (exponential)", "n": n, "us": round(us, 1),
                      "gb_per_s": round(gb / us * 1e6, 1)}))
    cl.shutdown()


if __name__ == "__main__":
    main()
