"""Debug: multi-step Cholesky at a given tile / n against LAPACK, timed."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_4886_b200 import distla, spawn

tile = int(sys.argv[1])
for n in [int(x) for x in sys.argv[2].split(",")]:
    rng = np.random.default_rng(n)
    B = rng.standard_normal((n, n))
    A = B @ B.T + n * np.eye(n)
    cl = spawn(1, tile=tile)
    t = time.perf_counter()
    try:
        C = distla.distribute(cl, "C", A, "triangular", distla.make_layout(n, cl.grid, h=1))
        L, _ = distla.distributed_cholesky(cl, C, "L")
        got = distla.collect(cl, L)
        err = np.linalg.norm(got - np.linalg.cholesky(A)) / np.linalg.norm(np.linalg.cholesky(A))
        print(f"tile {tile} n {n} T {(n + tile - 1) // tile}: relerr {err:.3e}  {time.perf_counter() - t:.2f} s", flush=True)
    except Exception as e:  # noqa
        print(f"tile {tile} n {n}: {type(e).__name__}: {e}  {time.perf_counter() - t:.2f} s", flush=True)
    cl.shutdown()
