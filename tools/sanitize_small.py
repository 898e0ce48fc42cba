"""Small runs of every dataflow kernel path under the checked build.

    make checked
    BGP_LIB_PATH=build/checked/libbgp.so python tools/sanitize_small.py

(compute-sanitizer is closed on this GPU pool; the checked build's BGP_CHECK
bounds / invariant checks trap on a bad tile coordinate, slot or gate.)

Covers: the single-GPU look-ahead factorization (update launches with the
in-launch POTRF / inverse / gated TRSM, both TRSM regimes, the tail
re-tiling) at tiles 128, 256 and 512; the kriging solve (bgp_trsm_rect
with its gated fused solve); the distributed sweep step (bgp_dist_step with
shadow tiles, the in-launch factor + solve and the panel push epilogue into
a destination buffer -- here this process's own) on a 1 x 1 grid, with the
gathered tail (parallel.factor_tail) at tile 256; the forward solve and the
covariance kernels.  Every result is checked against
numpy so a silent corruption fails the run too.
"""

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1305_4886_b200 import distla, spawn  # noqa: E402


def cov(n, seed):
    rng = np.random.default_rng(seed)
    X = rng.uniform(0, 1, (n, 2))
    d = np.sqrt(((X[:, None] - X[None]) ** 2).sum(-1))
    return np.exp(-d / 0.1) + 0.05 * np.eye(n)


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def check(name, err, tol):
    print(f"{name}: {err:.2e}", flush=True)
    if not err <= tol:
        raise SystemExit(f"{name} failed: {err} > {tol}")


class OwnExchange:
    """A panel 'exchange' whose only destination is this process's buffers:
    drives the push epilogue of bgp_dist_step without a peer."""

    def __init__(self, cl, tiles):
        import torch
        b = cl.tile
        self.tiles = tiles
        self.bufs = [torch.zeros((tiles, b, b), dtype=torch.float64, device=cl.device) for _ in range(2)]
        self.dst = [(ctypes.c_void_p * 1)(t.data_ptr()) for t in self.bufs]


def dist_sweep(cl, A):
    """dist_cholesky on a 1 x 1 grid through LibTileOps (step launches with
    the push epilogue) against LAPACK."""
    import torch

    from paper_1305_4886_b200.grid import DeviceGrid
    from paper_1305_4886_b200.parallel import LibTileOps, TileDist, dist_cholesky

    class Comm:
        world = 1

        def barrier_stream(self):
            pass

        def broadcast(self, t, src):
            pass

        def min_nonzero(self, v):
            return int(v)

        def all_gather(self, t):
            return [t]

    n, b = len(A), cl.tile
    td = TileDist(n, b, DeviceGrid(1), 0)
    T = td.T
    P = np.eye(T * b)
    P[:n, :n] = A
    local = torch.empty((td.storage_count, b, b), dtype=torch.float64, device=cl.device)
    for k, (I, J) in enumerate(td.storage_tiles):
        blk = P[I * b:(I + 1) * b, J * b:(J + 1) * b]
        local[k] = torch.from_numpy(np.ascontiguousarray((np.tril(blk) if I == J else blk).T))
    ops = LibTileOps(cl, n)
    xchg = OwnExchange(cl, T)
    ops.panel_exchange = lambda comm, T: xchg
    info = dist_cholesky(td, local, ops, Comm())
    assert info == 0, info
    L = np.zeros((T * b, T * b))
    for k, (I, J) in enumerate(td.tiles):
        L[I * b:(I + 1) * b, J * b:(J + 1) * b] = local[k].cpu().numpy().T
    return L[:n, :n]


def main():
    for tile in (128, 256, 512):
        cl = spawn(1, tile=tile)
        try:
            # look-ahead factorization: enough tiles for the large-step TRSM
            # regime at 128, the chain-bound (parallel pass) regime at all
            n = 9 * tile + 37
            A = cov(n, tile)
            lay = distla.make_layout(n, cl.grid)
            C = distla.distribute(cl, "C", A, "triangular", lay)
            L, _ = distla.distributed_cholesky(cl, C, "L")
            Lref = np.linalg.cholesky(A)
            check(f"potrf tile {tile}", relerr(distla.collect(cl, L), Lref), 1e-12)
            b = np.random.default_rng(1).standard_normal(n)
            bd = distla.distribute(cl, "b", b, "vector", lay)
            u = distla.triangular_solve(cl, L, bd, "u", side="forward")
            check(f"trsv tile {tile}", relerr(distla.collect(cl, u), np.linalg.solve(Lref, b)), 1e-12)
            m = tile + 61
            R = np.random.default_rng(2).standard_normal((n, m))
            Rd = distla.distribute(cl, "R", R, "rectangular", lay, distla.make_layout(m, cl.grid))
            V = distla.triangular_solve(cl, L, Rd, "V", side="forward")
            check(f"trsm_rect tile {tile}", relerr(distla.collect(cl, V), np.linalg.solve(Lref, R)), 1e-12)
            check(f"dist step tile {tile}", relerr(dist_sweep(cl, A), Lref), 1e-12)
            if tile == 256:  # enough tile rows for the gathered tail (24 at 256)
                At = cov(52 * 256 - 19, 7)
                check("dist step + gathered tail tile 256", relerr(dist_sweep(cl, At), np.linalg.cholesky(At)),
                      1e-12)
            # covariance kernels (fast interior path and the generic one)
            X = np.random.default_rng(3).uniform(0, 1, (n, 2))
            cl.push("inp", {"coords": X, "nu": 0.5})
            Cc = distla.construct_distributed(cl, "Cc", "triangular", "gen.matern-nugget.cov",
                                              [1.0, 0.1, 0.05], inputs_name="inp", row_layout=lay)
            d = np.sqrt(((X[:, None] - X[None]) ** 2).sum(-1))
            want = np.tril(np.exp(-d / 0.1) + 0.05 * np.eye(n))
            check(f"construct tile {tile}", np.abs(distla.collect(cl, Cc) - want).max(), 1e-14)
        finally:
            cl.shutdown()
    print("sanitize_small ok")


if __name__ == "__main__":
    main()
