"""The G > 1 code path end to end on the GPU box.

Two (or four) processes share cuda:0 and talk over gloo: every process drives
its own share of the 2-D block-cyclic tiles with the real libbgp tile kernels
(construct_tiles, tile_potrf, panel_trsm, the DMMA tile-list update,
tile_trsv, tile_gemv, tile_logdet).  No kernel waits on another process (all
exchanges are host-side gloo collectives), so sharing one GPU is safe.  On
an 8 x B200 box the same code runs with NCCL, one GPU per process.
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
        L, stats = distla.distributed_cholesky(cl, C, "L")
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
        out["owned"] = stats[0]["owned_blocks"]
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


@pytest.mark.parametrize("world,xfer", [(2, "push"), (4, "push"), (2, "nccl")])
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
        c = r["comm"]
        assert c["collectives"] > 0 and 0.0 <= c["exposed_comm_ms"] <= c["comm_ms"] + 1e-6
        assert abs(r["ll"] - want_ll) <= 1e-10 * abs(want_ll)
        assert relerr(r["mean"], want_mean) <= 1e-9
        assert relerr(r["se"], want_se) <= 1e-9
        assert relerr(r["pv"], want_pv) <= 1e-9
    lls = [r["ll"] for r in res.values()]
    assert all(v == lls[0] for v in lls)  # identical on every rank
