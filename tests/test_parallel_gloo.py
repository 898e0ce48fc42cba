"""Multi-GPU schedule (paper_1305_4886_b200/parallel.py) on CPU ranks over gloo.

The 2-D block-cyclic Cholesky, the distributed forward/back solves and the
rank-ordered log-det run here with world size 2 (1x2 grid), 4 (2x2 grid) and
8 (2x4 grid) on CPU processes, with both panel exchanges: the push (panel
buffers in shared memory, written by the solving rank) and the broadcast.  The collectives are real torch.distributed calls (gloo);
the tile arithmetic is a numpy/scipy stand-in (test-only), so what is
checked is the schedule: ownership, panel broadcasts, item lists, reduction
and solve order.  On GPUs the same functions drive libbgp over NCCL.
"""

import os
import socket

import numpy as np
import pytest
import scipy.linalg as la

from conftest import relerr, spd_matrix


class NumpyTileOps:
    """Tile kernels in numpy on torch CPU tensors (column-major tiles).

    Mirrors the device semantics the schedule relies on: a sweep step is
    the update of every listed tile, then (plan.diag) the factorization and
    inverse of the diagonal copy and the solve of the rank's panel tiles,
    each solved tile also copied into every rank's panel buffer (push); once
    a pivot failed, later steps are skipped (the device status)."""

    def __init__(self, b, n, xchg=None, tail=0):
        self.b, self.n = b, n
        self.xchg = xchg
        self.tail = tail
        self.info = 0

    def empty(self, shape):
        import torch
        return torch.zeros(shape, dtype=torch.float64)

    zeros = empty

    @staticmethod
    def _m(t):  # tile tensor (col-major storage) -> matrix view
        return t.numpy().T

    def potrf(self, local, k, row0):
        M = self._m(local[k])
        try:
            L = np.linalg.cholesky(np.tril(M) + np.tril(M, -1).T)
        except np.linalg.LinAlgError:
            return row0 + 1   # the stand-in reports the tile's first row
        M[:] = L
        return 0

    def begin(self):
        self.info = 0

    def end(self, info=0):
        return info or self.info

    def panel_exchange(self, comm, T):
        return self.xchg

    def sweep_begin(self, T):
        self.info = 0

    def tail_tiles(self, T):
        return self.tail

    def factor_tail(self, sub, T2, n2, row0):
        """The gathered trailing triangle, factored densely."""
        b = self.b
        tiles = [(I, J) for J in range(T2) for I in range(J, T2)]
        A = np.zeros((T2 * b, T2 * b))
        for t, (I, J) in enumerate(tiles):
            A[I * b:(I + 1) * b, J * b:(J + 1) * b] = self._m(sub[t])
        A = np.tril(A)
        try:
            L = np.linalg.cholesky(A + np.tril(A, -1).T)
        except np.linalg.LinAlgError:
            return row0 + 1
        for t, (I, J) in enumerate(tiles):
            self._m(sub[t])[:] = L[I * b:(I + 1) * b, J * b:(J + 1) * b]
        return 0

    def prepare_items(self, per_step):
        return [np.asarray(a).reshape(-1, 4) for a in per_step]

    def prepare_gemv_items(self, per_step):
        return [np.asarray(a).reshape(-1, 2) for a in per_step]

    def copy_tiles(self, dst, local, start, count):
        dst.copy_(local[start:start + count])

    def _factor_solve(self, local, d, row0, trsm, push):
        info = self.potrf(local, d, row0)
        if info:
            self.info = self.info or info
            return
        s, c = trsm
        if c == 0:
            return
        Li = np.linalg.inv(np.tril(self._m(local[d])))
        for t in range(s, s + c):
            M = self._m(local[t])
            M[:] = M @ Li.T
        if push is not None:
            xchg, which, slot0 = push
            for buf in xchg.dest[which]:
                buf[slot0:slot0 + c].copy_(local[s:s + c])

    def first_panel(self, local, d, trsm, push):
        if not self.info:
            self._factor_solve(local, d, 0, trsm, push)

    def step(self, J, local, panel, items, plan, par, push):
        if self.info:
            return
        for c, a, b, flags in items:
            M = self._m(local[c])
            U = self._m(panel[a]) @ self._m(panel[b]).T
            M[:] -= np.tril(U) if flags & 1 else U
        if plan.diag >= 0:
            self._factor_solve(local, plan.diag, plan.diag_row0, plan.trsm, push)

    def sub_into(self, out, a, b):
        out.copy_(a - b)

    def tile_trsv(self, local, k, row0, x, trans):
        L = np.tril(self._m(local[k]))
        xv = x.numpy()
        xv[:] = la.solve_triangular(L, xv, lower=True, trans=trans)
        return 0

    def gemv(self, local, items, xJ, acc, trans):
        a = acc.numpy()
        x = xJ.numpy()
        for k, tgt in items:
            M = self._m(local[k])
            a[tgt * self.b:(tgt + 1) * self.b] += (M.T @ x) if trans else (M @ x)

    def logdet_partial(self, local, diag):
        s = 0.0
        for k, J in diag:
            d = np.diag(self._m(local[k]))
            live = min(max(self.n - J * self.b, 0), self.b)
            s += 2.0 * float(np.sum(np.log(d[:live])))
        return s, 0


class SharedPanelExchange:
    """CPU stand-in of parallel.PanelExchange: every rank's two panel buffers
    live in shared memory (made by the test's parent process), so a push
    really writes into the other processes' buffers and the schedule's
    barriers are what keeps a rank from overwriting a panel a peer still
    reads."""

    def __init__(self, all_bufs, rank):
        # all_bufs[r][w]: rank r's buffer w, (tiles, b, b)
        self.bufs = list(all_bufs[rank])
        self.dest = [[all_bufs[r][w] for r in range(len(all_bufs))] for w in range(2)]
        self.tiles = self.bufs[0].shape[0]


def _local_tiles(td, P, b):
    """This rank's tile stack (owned tiles, then shadow diagonal tiles) of
    the padded dense matrix P."""
    import torch
    st = td.storage_tiles
    local = torch.zeros((len(st), b, b), dtype=torch.float64)
    for k, (I, J) in enumerate(st):
        blk = P[I * b:(I + 1) * b, J * b:(J + 1) * b]
        local[k].numpy().T[:] = np.tril(blk) if I == J else blk
    return local


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, b, q, bufs, tail=0):
    import torch
    import torch.distributed as dist

    from paper_1305_4886_b200.grid import DeviceGrid
    from paper_1305_4886_b200.parallel import (TileDist, TorchComm, dist_cholesky,
                                               dist_logdet, dist_trsv)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = spd_matrix(n, seed=n)
        T = -(-n // b)
        P = np.zeros((T * b, T * b))
        P[:n, :n] = A
        for t in range(n, T * b):
            P[t, t] = 1.0
        td = TileDist(n, b, DeviceGrid(world), rank)
        local = _local_tiles(td, P, b)
        xchg = SharedPanelExchange(bufs, rank) if bufs is not None else None
        ops, comm = NumpyTileOps(b, n, xchg, tail), TorchComm()
        info = dist_cholesky(td, local, ops, comm)
        # gather L into a dense matrix on every rank
        Ld = torch.zeros((T * b, T * b), dtype=torch.float64)
        for k, (I, J) in enumerate(td.tiles):
            Ld[I * b:(I + 1) * b, J * b:(J + 1) * b] = torch.from_numpy(local[k].numpy().T.copy())
        dist.all_reduce(Ld)
        # the shadow copies of the diagonal tiles factor to the owner's L
        # (those of the gathered tail are not used)
        J0 = T - tail if 0 < tail and 2 * tail < T else T
        shadow_ok = all(np.array_equal(np.tril(local[td.shadow_local[K]].numpy().T),
                                       Ld.numpy()[K * b:(K + 1) * b, K * b:(K + 1) * b])
                        for K in td.shadows if K < J0)
        ops.xchg = None
        y = torch.zeros(T * b, dtype=torch.float64)
        y[:n] = torch.from_numpy(np.random.default_rng(3).standard_normal(n))
        u, info_f = dist_trsv(td, local, y, ops, comm, forward=True)
        x, info_b = dist_trsv(td, local, u, ops, comm, forward=False)
        ld, info_l = dist_logdet(td, local, ops, comm)
        q.put((rank, info, info_f, info_b, info_l, np.tril(Ld.numpy()[:n, :n]), u.numpy()[:n].copy(),
               x.numpy()[:n].copy(), ld, td.count, shadow_ok))
    finally:
        dist.destroy_process_group()


def _shared_bufs(world, n, b):
    import torch
    T = -(-n // b)
    out = []
    for _ in range(world):
        pair = []
        for _ in range(2):
            t = torch.full((max(T, world), b, b), float("nan"), dtype=torch.float64)
            t.share_memory_()
            pair.append(t)
        out.append(pair)
    return out


@pytest.mark.parametrize("xfer", ["push", "broadcast"])
@pytest.mark.parametrize("world,n,b,tail", [(2, 37, 8, 0), (2, 100, 16, 0), (4, 90, 8, 3), (4, 37, 16, 0),
                                            (8, 100, 8, 4), (8, 61, 4, 0)])
def test_distributed_cholesky_solves_logdet(world, n, b, tail, xfer):
    """tail > 0: the last `tail` tile rows are gathered to every rank and
    finished there (parallel.factor_tail)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    bufs = _shared_bufs(world, n, b) if xfer == "push" else None
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, b, q, bufs, tail)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = spd_matrix(n, seed=n)
    y = np.random.default_rng(3).standard_normal(n)
    Lref = np.linalg.cholesky(A)
    T = -(-n // b)
    assert sum(o[9] for o in out) == T * (T + 1) // 2      # tiles partitioned
    for rank, info, info_f, info_b, info_l, L, u, x, ld, _, shadow_ok in out:
        assert info == info_f == info_b == info_l == 0
        assert shadow_ok
        assert relerr(L, Lref) <= 1e-12
        assert relerr(u, np.linalg.solve(Lref, y)) <= 1e-12
        assert relerr(x, np.linalg.solve(A, y)) <= 1e-10
        assert abs(ld - np.linalg.slogdet(A)[1]) <= 1e-12 * abs(ld)
    # every rank agrees bit for bit on the replicated results
    for o in out[1:]:
        np.testing.assert_array_equal(o[6], out[0][6])
        assert o[8] == out[0][8]


def _fail_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1305_4886_b200.grid import DeviceGrid
    from paper_1305_4886_b200.parallel import TileDist, TorchComm, dist_cholesky
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, b = 24, 8
        A = -np.eye(n)
        A[:8, :8] = spd_matrix(8, seed=1)     # block 0 fine, block 1 fails
        td = TileDist(n, b, DeviceGrid(world), rank)
        info = dist_cholesky(td, _local_tiles(td, A, b), NumpyTileOps(b, n), TorchComm())
        q.put(info)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_failure_is_agreed_by_all_ranks(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fail_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    infos = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert infos == [9] * world   # first row of tile 1 (1-based)


def test_tile_dist_layout_invariants():
    from paper_1305_4886_b200.grid import DeviceGrid
    from paper_1305_4886_b200.parallel import TileDist
    for G in (1, 2, 4, 8):
        T = 13
        dists = [TileDist(T * 4, 4, DeviceGrid(G), r) for r in range(G)]
        allt = sorted((int(I), int(J)) for d in dists for I, J in d.tiles)
        assert allt == sorted((I, J) for J in range(T) for I in range(J, T))
        for J in range(T - 1):
            chunks, slot, ntot = dists[0].panel_layout(J)
            assert ntot == T - J - 1
            assert sorted(slot[J + 1:]) == list(range(ntot))
            for root, off, cnt in chunks:
                s, c = dists[root].my_panel(J)
                assert c == cnt
                assert [int(I) for I in dists[root].tiles[s:s + c, 0]] == \
                       [I for I in range(J + 1, T) if slot[I] >= off and slot[I] < off + cnt]
            # step plans: every rank holding panel-(J+1) tiles factors a
            # copy of (J+1, J+1); gates cover exactly its column-(J+1) items
            for r, d in enumerate(dists):
                plan = d.step_plan(J, slot)
                ps, pc_ = d.my_panel(J + 1)
                assert plan.trsm == ((ps, pc_) if plan.diag >= 0 else (ps, 0))
                if pc_:
                    assert plan.diag >= 0
                if d.owner(J + 1, J + 1) == r:
                    assert plan.diag == d.local[(J + 1, J + 1)]
                gates = plan.items[:, 3] >> 8
                assert (gates[:plan.col_items] > 0).all() and (gates[plan.col_items:] == 0).all()
                if plan.diag >= 0:
                    assert sorted(gates[:plan.col_items] - 1) == list(range(1 + plan.trsm[1]))


def test_col_shards_partition():
    from paper_1305_4886_b200.parallel import col_shards
    for T in (0, 1, 3, 8, 13, 32):
        for G in (1, 2, 4, 8):
            sh = col_shards(T, G)
            assert len(sh) == G and sh[0][0] == 0 and sh[-1][1] == T
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            widths = [r1 - r0 for r0, r1 in sh]
            assert max(widths) - min(widths) <= 1


def _rhs_worker(rank, world, port, q):
    """Kriging solve with RHS columns sharded over ranks (ops.solve_rect at
    G > 1): each rank solves its tile-row shard of the transposed RHS
    (Tn, Tm, b, b) storage, then the shards are all-gathered."""
    import torch
    import torch.distributed as dist

    from paper_1305_4886_b200.parallel import TorchComm, col_shards, gather_col_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m, b = 40, 37, 8
        Tn, Tm = -(-n // b), -(-m // b)
        L = np.linalg.cholesky(spd_matrix(n, seed=2))
        B = np.random.default_rng(7).standard_normal((n, m))
        # transposed storage: tile (I, J) of B^T (m x n) at J*Tm + I, column-major inside
        Bt = np.zeros((Tm * b, Tn * b))
        Bt[:m, :n] = B.T
        tiles = torch.zeros((Tn, Tm, b, b), dtype=torch.float64)
        for J in range(Tn):
            for I in range(Tm):
                tiles[J, I] = torch.from_numpy(Bt[I * b:(I + 1) * b, J * b:(J + 1) * b].T.copy())
        shards = col_shards(Tm, world)
        r0, r1 = shards[rank]
        mine = tiles[:, r0:r1].clone()
        # local solve of my columns: X^T = B^T L^-T on the dense shard
        cols = Bt[r0 * b:r1 * b, :n]
        sol = np.linalg.solve(L, cols.T).T
        for J in range(Tn):
            for I in range(r1 - r0):
                blk = np.zeros((b, b))
                piece = sol[I * b:(I + 1) * b, J * b:(J + 1) * b]
                blk[:piece.shape[0], :piece.shape[1]] = piece
                mine[J, I] = torch.from_numpy(blk.T.copy())
        width = max(s1 - s0 for s0, s1 in shards)
        part = torch.zeros((Tn, width, b, b), dtype=torch.float64)
        part[:, :r1 - r0] = mine
        full = torch.zeros_like(tiles)

        def fill(s0, s1, piece):
            full[:, s0:s1] = piece
        gather_col_shards(TorchComm(), part, shards, fill)
        Xt = np.zeros((Tm * b, Tn * b))
        for J in range(Tn):
            for I in range(Tm):
                Xt[I * b:(I + 1) * b, J * b:(J + 1) * b] = full[J, I].numpy().T
        q.put((rank, Xt[:m, :n].T.copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_rhs_solve_gathers_full_result(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rhs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    L = np.linalg.cholesky(spd_matrix(40, seed=2))
    B = np.random.default_rng(7).standard_normal((40, 37))
    want = np.linalg.solve(L, B)
    for _, X in out:
        assert relerr(X, want) <= 1e-12


def test_exposed_time_intervals():
    from paper_1305_4886_b200.parallel import exposed_time
    assert exposed_time([], [(0, 5)]) == 0
    assert exposed_time([(0, 2)], []) == 2
    assert exposed_time([(1, 2)], [(0, 5)]) == 0                 # fully hidden
    assert exposed_time([(4, 7)], [(0, 5)]) == 2                 # tail exposed
    assert exposed_time([(0, 10)], [(1, 2), (2, 4), (6, 7)]) == 6  # merged cover
    assert exposed_time([(0, 3), (5, 9)], [(2, 6), (8, 20)]) == 2 + 2
