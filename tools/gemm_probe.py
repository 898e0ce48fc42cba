"""Time the trailing-update GEMM (list mode, one Cholesky step of k tiles) for
each libbgp variant given on the command line, e.g. probe builds made with
-DBGP_EXP_NO_TMA / -DBGP_EXP_NO_EPI (see tools/gemm_probe.sh).

    python tools/gemm_probe.py lib1.so [lib2.so ...]
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1305_4886_b200 import _lib  # noqa: E402


def main():
    b = int(os.environ.get("PROBE_B", "256"))
    T = int(os.environ.get("PROBE_T", str(96 * 256 // b)))
    reps = int(os.environ.get("PROBE_REPS", "5"))
    dev = torch.device("cuda:0")
    nt = T * (T + 1) // 2
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    tiles = torch.randn((nt, b, b), dtype=torch.float64, device=dev, generator=g) * 1e-3

    def tri(I, J):
        return J * T - J * (J - 1) // 2 + (I - J)

    items = []
    for C in range(1, T):
        for R in range(C, T):
            items.append((tri(R, C), tri(R, 0), tri(C, 0), int(R == C)))
    it = torch.tensor(np.array(items, dtype=np.int32).ravel(), device=dev)
    k = T - 1
    flops = b ** 3 * k * k
    s = torch.cuda.current_stream().cuda_stream
    for path in sys.argv[1:]:
        lib = _lib.load(os.path.abspath(path))
        ctx = ctypes.c_void_p()
        assert lib.bgp_init(0, ctypes.byref(ctx)) == 0
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        run = lambda: lib.bgp_tile_update(ctx, p(tiles), p(tiles), p(tiles), p(it), len(items), b, s)  # noqa: E731
        assert run() == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        print(json.dumps({"lib": os.path.basename(path), "trailing_tiles": k, "us": round(us, 1),
                          "tflops": round(flops / us / 1e6, 2)}), flush=True)
        # item-length sweep: S = V^T V with Tn k-tiles per output block
        if os.environ.get("PROBE_XPROD"):
            for Tm, Tn in ((96, 1), (64, 2), (48, 4), (32, 8)):
                V = torch.randn((Tn, Tm, b, b), dtype=torch.float64, device=dev, generator=g)
                S = torch.empty((Tm * (Tm + 1) // 2, b, b), dtype=torch.float64, device=dev)
                f = lambda: lib.bgp_xprod_self(ctx, p(V), Tn * b, Tm * b, b, p(S), s)  # noqa: E731
                assert f() == 0
                torch.cuda.synchronize()
                e0.record()
                for _ in range(reps):
                    f()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / reps * 1e3
                fl = 2.0 * b ** 3 * Tn * Tm * (Tm + 1) / 2
                print(json.dumps({"lib": os.path.basename(path), "xprod_Tm": Tm, "k_tiles": Tn,
                                  "us": round(us, 1), "tflops": round(fl / us / 1e6, 2)}), flush=True)
                del V, S
        if hasattr(lib, "bgp_probe_trace"):
            buf = np.zeros((148, 2, 64, 6), dtype=np.uint64)
            lib.bgp_probe_trace(ctypes.c_void_p(buf.ctypes.data))
            np.save(os.path.join(ROOT, "gpurun_out", "probe", "trace_" + os.path.basename(path)[:-3] + ".npy"), buf)
        if hasattr(lib, "bgp_probe_strace"):
            buf = np.zeros((148, 2, 64, 20), dtype=np.uint64)
            lib.bgp_probe_strace(ctypes.c_void_p(buf.ctypes.data))
            np.save(os.path.join(ROOT, "gpurun_out", "probe", "strace_" + os.path.basename(path)[:-3] + ".npy"), buf)
        lib.bgp_finalize(ctx)


if __name__ == "__main__":
    main()
