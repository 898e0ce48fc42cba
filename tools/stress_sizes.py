"""Robustness sweep of the factorization schedules (look-ahead launches, the
multi-step tail launch, the fused first panel, tail re-tiling): many sizes
at every tile, one cluster per tile, each factor against LAPACK.

    python tools/stress_sizes.py [reps] > out.txt     (GPU)

Prints one line per factorization and a final summary line."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_4886_b200 import distla, spawn  # noqa: E402


def cov(n, seed):
    rng = np.random.default_rng(seed)
    X = rng.uniform(0, 1, (n, 2))
    d = np.sqrt(((X[:, None] - X[None]) ** 2).sum(-1))
    return np.exp(-d / 0.1) + 0.02 * np.eye(n)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    rng = np.random.default_rng(12345)
    worst, count, bad = 0.0, 0, 0
    for tile in (128, 256, 384, 512):
        cl = spawn(1, tile=tile)
        sizes = sorted(set([1, 2, tile - 1, tile, tile + 1, 2 * tile, 3 * tile - 5]
                           + [int(v) for v in rng.integers(3, 9000, size=12)]))
        for rep in range(reps):
            for n in sizes:
                A = cov(n, n + rep)
                C = distla.distribute(cl, "C", A, "triangular", distla.make_layout(n, cl.grid, h=2))
                L, _ = distla.distributed_cholesky(cl, C, "L")
                got = distla.collect(cl, L)
                want = np.linalg.cholesky(A)
                err = np.linalg.norm(got - want) / np.linalg.norm(want)
                worst = max(worst, err)
                count += 1
                bad += err > 1e-12
                print(f"tile {tile} n {n} rep {rep}: relerr {err:.2e}", flush=True)
                cl.remote_rm("L")
        cl.shutdown()
    print(f"SUMMARY factorizations {count} worst relerr {worst:.2e} over 1e-12: {bad}")


if __name__ == "__main__":
    main()
