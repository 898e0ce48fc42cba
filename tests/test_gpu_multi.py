"""The G > 1 code path end to end on the GPU box.

Two, four or eight processes share cuda:0 and talk over gloo: every process
drives its own share of the 2-D block-cyclic tiles (plus its shadow diagonal
tiles) with the real libbgp kernels (construct_tiles, the one-launch sweep
step bgp_dist_step with its in-launch POTRF / inverse / panel solve + push,
tile_trsv, tile_gemv, tile_logdet).  No kernel waits on another process (the
steps are ordered by host-side gloo barriers), so sharing one GPU is safe.
On an 8 x B200 box the same code runs with NCCL, one GPU per process.
test_master_spawn_* drive the same path through spawn(P) from this process
(transport.master: P worker processes, per-rank results in rank order).
"""

import os
import socket

import numpy as np
import pytest

from conftest import relerr, spd_matrix

pytestmark = pytest.mark.gpu

# 23 x 23 = 529 prediction points: 5 tile columns of 128, so the kriging
# RHS shards are uneven (3 + 2 on two ranks; 2, 1, 1, 1 on four)
PRED_SIDE = 23


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, xfer="push"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK="0", BGP_PANEL_XFER=xfer)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import blockgp_oracle as orc
        from paper_1305_4886_b200 import distla, spawn
        from paper_1305_4886_b200.errors import NotPositiveDefinite
        from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
        cl = spawn(world, tile=128, device=0)
        out = {}
        # distla on a random SPD matrix (distribute -> cholesky -> solves -> logdet)
        n = 700
        A = spd_matrix(n, seed=5)
        lay = distla.make_layout(n, cl.grid, h=2)
        C = distla.distribute(cl, "C", A, "triangular", lay)
        cl.comm_timeline = True  # CUDA-event spans of broadcasts and updates
        launches = cl.launches()
        L, stats = distla.distributed_cholesky(cl, C, "L")
        out["chol_launches"] = cl.launches() - launches
        cl.comm_timeline = False
        out["comm"] = cl.last_comm
        x = cl.__dict__.get("_panel_xchg", {}).get("x")
        out["xfer"] = "push" if (x is not None and x.ok) else "nccl"
        out["L"] = distla.collect(cl, L)
        bvec = np.random.default_rng(5).standard_normal(n)
        bd = distla.distribute(cl, "b", bvec, "vector", lay)
        u = distla.triangular_solve(cl, L, bd, "u", side="forward")
        x = distla.triangular_solve(cl, L, u, "x", side="back")
        out["x"] = distla.collect(cl, x)
        out["logdet"] = distla.log_det_from_chol(cl, L)
        assert len(stats) == world  # per-rank stats, gathered
        out["owned"] = stats[rank]["owned_tiles"]
        # NotPositiveDefinite is agreed by every rank and leaves no factor
        Cn = distla.distribute(cl, "Cn", -np.eye(300), "triangular", distla.make_layout(300, cl.grid, h=1))
        try:
            distla.distributed_cholesky(cl, Cn, "Ln")
            out["npd"] = None
        except NotPositiveDefinite as exc:
            out["npd"] = exc.block_index
        out["ls"] = cl.remote_ls(1)
        # GP log density + kriging (config-1 recipe at n = 900)
        kern, X, theta, extra, z = orc.config_inputs(1, n=900)
        y = np.linalg.cholesky(orc.dense_cov(kern, theta, X, **extra)) @ z
        Xp = orc.c3_pred_coords(PRED_SIDE)
        prob = KrigeProblem(cl, "g", builtin_spec(kern, X, Xp, **extra), y, theta, m=len(Xp))
        out["ll"] = prob.log_density()
        out["mean"], out["se"] = prob.predict(se_fit=True)
        out["pv"] = prob.prediction_variance()
        cl.shutdown()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,xfer", [(2, "push"), (4, "push"), (8, "push"), (2, "nccl")])
def test_multi_rank_path_on_one_gpu(world, xfer):
    """xfer "push": the panel TRSM stores into every rank's IPC-mapped panel
    buffer (bgp_panel_trsm_push; here all mappings are on cuda:0); "nccl":
    TRSM, then broadcasts of the panel chunks."""
    import torch.multiprocessing as mp
    from oracle import blockgp_oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, xfer)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    import queue
    import time
    t0 = time.time()
    while len(res) < world:
        try:
            rank, out = q.get(timeout=2)
            res[rank] = out
        except queue.Empty:
            dead = [p for p in procs if p.exitcode not in (None, 0)]
            if dead or time.time() - t0 > 400:
                for p in procs:
                    p.kill()
                pytest.fail(f"worker failed (exit codes {[p.exitcode for p in procs]})")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 700
    A = spd_matrix(n, seed=5)
    bvec = np.random.default_rng(5).standard_normal(n)
    kern, X, theta, extra, z = orc.config_inputs(1, n=900)
    y = np.linalg.cholesky(orc.dense_cov(kern, theta, X, **extra)) @ z
    ref = orc.OracleProblem(kern, X, y, theta, pred_coords=orc.c3_pred_coords(PRED_SIDE), **extra)
    want_ll = ref.log_density()
    want_mean, want_se = ref.predict(se_fit=True)
    want_pv = ref.prediction_variance()
    T = -(-n // 128)
    assert sum(r["owned"] for r in res.values()) == T * (T + 1) // 2
    for r in res.values():
        assert relerr(r["L"], np.linalg.cholesky(A)) <= 1e-12
        assert relerr(r["x"], np.linalg.solve(A, bvec)) <= 1e-10
        assert abs(r["logdet"] - np.linalg.slogdet(A)[1]) <= 1e-12 * abs(r["logdet"])
        assert r["npd"] == 1 and "Ln" not in r["ls"] and "Cn" not in r["ls"]
        assert r["xfer"] == xfer
        # the panel solve and its exchange run inside the step launches: one
        # launch per step (+ panel 0's factor and solve), nothing on the side
        assert r["chol_launches"] <= T + 1
        assert len(r["comm"]["step_launch_ms"]) <= T - 1
        c = r["comm"]
        assert c["collectives"] > 0 and 0.0 <= c["exposed_comm_ms"] <= c["comm_ms"] + 1e-6
        assert abs(r["ll"] - want_ll) <= 1e-10 * abs(want_ll)
        assert relerr(r["mean"], want_mean) <= 1e-9
        assert relerr(r["se"], want_se) <= 1e-9
        assert relerr(r["pv"], want_pv) <= 1e-9
    lls = [r["ll"] for r in res.values()]
    assert all(v == lls[0] for v in lls)  # identical on every rank


def test_master_spawn_reference_call_sequence():
    """The reference's call sequence unchanged at P = 2 from a plain process:
    spawn(2) -> KrigeProblem(...).log_density() / predict, distla calls with
    P-length per-rank results (bg/transport/base.py:213-234)."""
    from oracle import blockgp_oracle as orc
    from paper_1305_4886_b200 import distla, spawn
    from paper_1305_4886_b200.errors import NotPositiveDefinite
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    cl = spawn(2, tile=128, devices=[0, 0])
    try:
        assert cl.P == 2 and cl.comm_backend == "gloo"
        n = 500
        A = spd_matrix(n, seed=9)
        lay = distla.make_layout(n, cl.grid, h=2)
        C = distla.distribute(cl, "C", A, "triangular", lay)
        L, stats = distla.distributed_cholesky(cl, C, "L")
        assert len(stats) == 2
        T = -(-n // 128)
        assert sum(s["owned_tiles"] for s in stats) == T * (T + 1) // 2
        assert relerr(distla.collect(cl, L), np.linalg.cholesky(A)) <= 1e-12
        parts = cl.run("distla.logdet", l_name="L")
        assert len(parts) == 2
        assert abs(sum(parts) - np.linalg.slogdet(A)[1]) <= 1e-12 * abs(sum(parts))
        with pytest.raises(NotPositiveDefinite) as ei:
            Cn = distla.distribute(cl, "Cn", -np.eye(300), "triangular",
                                   distla.make_layout(300, cl.grid, h=1))
            distla.distributed_cholesky(cl, Cn, "Ln")
        assert ei.value.block_index == 1 and "Ln" not in cl.remote_ls()
        kern, X, theta, extra, z = orc.config_inputs(1, n=700)
        y = np.linalg.cholesky(orc.dense_cov(kern, theta, X, **extra)) @ z
        Xp = orc.c3_pred_coords(12)
        prob = KrigeProblem(cl, "g", builtin_spec(kern, X, Xp, **extra), y, theta, m=len(Xp))
        ll = prob.log_density()
        mean, se = prob.predict(se_fit=True)
        assert len(prob.last_cholesky_stats) == 2
    finally:
        cl.shutdown()
    ref = orc.OracleProblem(kern, X, y, theta, pred_coords=Xp, **extra)
    want = ref.log_density()
    rmean, rse = ref.predict(se_fit=True)
    assert abs(ll - want) <= 1e-10 * abs(want)
    assert relerr(mean, rmean) <= 1e-9 and relerr(se, rse) <= 1e-9
    assert cl.state == "shutdown"


class _OwnExchange:
    """A panel exchange whose only destination is this process's buffers."""

    def __init__(self, cl, tiles):
        import ctypes

        import torch
        self.tiles = tiles
        self.bufs = [torch.zeros((tiles, cl.tile, cl.tile), dtype=torch.float64, device=cl.device)
                     for _ in range(2)]
        self.dst = [(ctypes.c_void_p * 1)(t.data_ptr()) for t in self.bufs]


class _OneRank:
    world = 1

    def barrier_stream(self):
        pass

    def broadcast(self, t, src):
        pass

    def min_nonzero(self, v):
        return int(v)

    def all_gather(self, t):
        return [t]


@pytest.mark.parametrize("tile,nt", [(128, 11), (256, 5), (512, 3), (256, 52), (512, 27)])
@pytest.mark.parametrize("push", [True, False])
def test_dist_sweep_steps_in_one_process(cluster_factory, tile, nt, push):
    """The sweep-step launch (bgp_dist_step: update + in-launch POTRF /
    inverse / gated TRSM, with or without the push epilogue) driven by
    dist_cholesky on a 1 x 1 grid, against LAPACK; with nt > 2 x the tail
    (24 / 12 tile rows at 256 / 512) the last rows go through the gathered
    tail (parallel.factor_tail, re-tiled to 128)."""
    import torch

    from paper_1305_4886_b200.grid import DeviceGrid
    from paper_1305_4886_b200.parallel import LibTileOps, TileDist, dist_cholesky
    cl = cluster_factory(tile=tile)
    n = nt * tile - 19
    if n <= 4000:
        A = spd_matrix(n, seed=tile)
    else:  # a covariance matrix: cheap to build at this size
        X = np.random.default_rng(tile).uniform(0, 1, (n, 2))
        A = np.exp(-np.sqrt(((X[:, None] - X[None]) ** 2).sum(-1)) / 0.2) + 0.1 * np.eye(n)
    td = TileDist(n, tile, DeviceGrid(1), 0)
    T = td.T
    P = np.eye(T * tile)
    P[:n, :n] = A
    local = torch.empty((td.storage_count, tile, tile), dtype=torch.float64, device=cl.device)
    for k, (I, J) in enumerate(td.storage_tiles):
        blk = P[I * tile:(I + 1) * tile, J * tile:(J + 1) * tile]
        local[k] = torch.from_numpy(np.ascontiguousarray((np.tril(blk) if I == J else blk).T))
    ops = LibTileOps(cl, n)
    xchg = _OwnExchange(cl, T) if push else None
    ops.panel_exchange = lambda comm, T: xchg
    launches = cl.launches()
    assert dist_cholesky(td, local, ops, _OneRank()) == 0
    tail = ops.tail_tiles(T)
    if 2 * tail >= T:  # one launch per step (+ the first panel)
        assert cl.launches() - launches <= T + 2
    L = np.zeros((T * tile, T * tile))
    for k, (I, J) in enumerate(td.tiles):
        L[I * tile:(I + 1) * tile, J * tile:(J + 1) * tile] = local[k].cpu().numpy().T
    assert relerr(L[:n, :n], np.linalg.cholesky(A)) <= 1e-12


def _tail_worker(rank, world, port, q, n):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK="0")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import blockgp_oracle as orc
        from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
        from paper_1305_4886_b200 import spawn
        kern, X, theta, extra, z = orc.config_inputs(4, n=n)
        cl = spawn(world, tile=256, device=0)
        prob = KrigeProblem(cl, "t", builtin_spec(kern, X, **extra), z, theta)
        q.put((rank, prob.log_density()))
        cl.shutdown()
    finally:
        dist.destroy_process_group()


def test_distributed_sweep_with_gathered_tail_two_ranks():
    """2 ranks on one GPU at a size where the sweep's last 24 tile rows of
    256 are gathered and finished on every rank (parallel.factor_tail): the
    log-density equals the single-GPU path's."""
    import torch.multiprocessing as mp
    from oracle import blockgp_oracle as orc
    from paper_1305_4886_b200 import spawn
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    n = 52 * 256 - 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tail_worker, args=(r, 2, port, q, n)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    kern, X, theta, extra, z = orc.config_inputs(4, n=n)
    cl = spawn(1, tile=256)
    try:
        want = KrigeProblem(cl, "t", builtin_spec(kern, X, **extra), z, theta).log_density()
    finally:
        cl.shutdown()
    assert out[0] == out[1]
    assert abs(out[0] - want) <= 1e-10 * abs(want)
