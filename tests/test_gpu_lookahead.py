"""Multi-step tile Cholesky on the GPU: the look-ahead pipeline (POTRF of the
next panel on a side stream, gated by the trailing update) and the panel TRSM
on the DMMA GEMM (in-place passes with the tile inverse) against LAPACK.

The reference's checks (pkg/tests/test_distla.py:92-141: vs
np.linalg.cholesky <= 1e-12, NotPositiveDefinite block index, no partial
factor left behind) at sizes with five or more tile columns, so every
pipeline stage runs several times, for every supported tile size.
"""

import numpy as np
import pytest

from conftest import relerr, spd_matrix

pytestmark = pytest.mark.gpu


def _cov(n, seed):
    """C4-style covariance: exponential kernel, 10 % near-duplicates, nugget."""
    rng = np.random.default_rng(seed)
    X = rng.uniform(0, 1, (n, 2))
    dup = rng.choice(n, n // 10, replace=False)
    X[dup[1:]] = X[dup[:-1]] + 1e-4 * rng.standard_normal((len(dup) - 1, 2))
    d = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    return np.exp(-d / 0.08) + 0.02 * np.eye(n)


@pytest.mark.parametrize("tile,ntiles", [(128, 9), (256, 6), (384, 6), (512, 5)])
def test_lookahead_matches_lapack(cluster_factory, tile, ntiles):
    from paper_1305_4886_b200 import distla
    n = tile * ntiles - 37  # ragged last tile
    cl = cluster_factory(tile=tile)
    for A in (spd_matrix(n, seed=tile), _cov(n, seed=tile)):
        C = distla.distribute(cl, "C", A, "triangular", distla.make_layout(n, cl.grid, h=3))
        L, _ = distla.distributed_cholesky(cl, C, "L")
        got = distla.collect(cl, L)
        want = np.linalg.cholesky(A)
        assert relerr(got, want) <= 1e-12
        assert relerr(got @ got.T, A) <= 1e-13
        cl.remote_rm("L")


@pytest.mark.parametrize("tile", [128, 256])
def test_lookahead_late_failure(cluster_factory, tile):
    """A non-positive pivot in a late panel (factored on the look-ahead
    stream) raises NotPositiveDefinite for the right block and leaves neither
    the input nor a partial factor behind."""
    from paper_1305_4886_b200 import distla
    from paper_1305_4886_b200.errors import NotPositiveDefinite
    n = tile * 6
    A = spd_matrix(n, seed=3)
    bad = 4 * tile + 5  # 0-based row inside tile column 4
    A[bad, bad] = -1.0
    cl = cluster_factory(tile=tile)
    lay = distla.make_layout(n, cl.grid, h=6)
    C = distla.distribute(cl, "C", A, "triangular", lay)
    with pytest.raises(NotPositiveDefinite) as info:
        distla.distributed_cholesky(cl, C, "L")
    assert info.value.block_index == bad // lay.block_size + 1
    names = set(cl.remote_ls())
    assert "C" not in names and "L" not in names
    # the pipeline recovers: the next factorization on the same cluster works
    A2 = spd_matrix(n, seed=4)
    C2 = distla.distribute(cl, "C2", A2, "triangular", lay)
    L2, _ = distla.distributed_cholesky(cl, C2, "L2")
    assert relerr(distla.collect(cl, L2), np.linalg.cholesky(A2)) <= 1e-12


@pytest.mark.parametrize("tile", [128, 256, 384, 512])
def test_tile_inverse(cluster_factory, tile):
    """The one-CTA block-diagonal inverse the fused panel TRSM uses."""
    import ctypes
    import torch
    cl = cluster_factory(tile=tile)
    A = spd_matrix(tile, seed=tile)
    t = torch.from_numpy(np.tril(A).T.copy()).to(cl.device)  # column-major lower tile
    linv = torch.empty_like(t)
    info = ctypes.c_int64()
    rc = cl.lib.bgp_tile_potrf_inv(cl._ctx, ctypes.c_void_p(t.data_ptr()), tile,
                                   ctypes.c_void_p(linv.data_ptr()), ctypes.byref(info), cl.stream)
    assert rc == 0 and info.value == 0
    L = np.linalg.cholesky(A)
    got = linv.cpu().numpy().T  # column-major -> row-major
    assert relerr(got, np.linalg.inv(L)) <= 1e-12
    assert np.all(np.triu(got, 1) == 0.0)


@pytest.mark.parametrize("tail,n", [(2, 512 * 7 - 100), (3, 512 * 9 - 7), (4, 512 * 9)])
def test_tail_retiling_matches_lapack(cluster_factory, tail, n):
    """512-tile factorization whose last `tail` tile rows are re-tiled to 256."""
    from paper_1305_4886_b200 import distla
    cl = cluster_factory(tile=512)
    assert cl.lib.bgp_set_tail(cl._ctx, tail) == 0
    for A in (spd_matrix(n, seed=n), _cov(n, seed=n)):
        C = distla.distribute(cl, "C", A, "triangular", distla.make_layout(n, cl.grid, h=2))
        L, _ = distla.distributed_cholesky(cl, C, "L")
        got = distla.collect(cl, L)
        assert relerr(got, np.linalg.cholesky(A)) <= 1e-12
        assert abs(distla.log_det_from_chol(cl, L) - np.linalg.slogdet(A)[1]) <= 1e-10 * abs(np.linalg.slogdet(A)[1])
        cl.remote_rm("L")


def test_tail_failure_row(cluster_factory):
    """A non-positive pivot inside the re-tiled tail reports its global row."""
    from paper_1305_4886_b200 import distla
    from paper_1305_4886_b200.errors import NotPositiveDefinite
    n = 512 * 7
    A = spd_matrix(n, seed=9)
    bad = 512 * 6 + 300  # inside the last two tile rows (tail = 2)
    A[bad, bad] = -1.0
    cl = cluster_factory(tile=512)
    cl.lib.bgp_set_tail(cl._ctx, 2)
    lay = distla.make_layout(n, cl.grid, h=7)
    C = distla.distribute(cl, "C", A, "triangular", lay)
    with pytest.raises(NotPositiveDefinite) as info:
        distla.distributed_cholesky(cl, C, "L")
    assert info.value.block_index == bad // lay.block_size + 1


def test_large_steps_keep_serial_passes(cluster_factory):
    """Steps with more trailing tiles than the chain-bound threshold (48 at
    tile 128) run a slab's TRSM passes as one task; smaller ones as parallel
    tasks.  n = 56 tiles of 128 covers both regimes in one factorization."""
    from paper_1305_4886_b200 import distla
    n = 128 * 56 - 5
    cl = cluster_factory(tile=128)
    A = _cov(n, seed=11)
    C = distla.distribute(cl, "C", A, "triangular", distla.make_layout(n, cl.grid, h=4))
    L, _ = distla.distributed_cholesky(cl, C, "L")
    got = distla.collect(cl, L)
    assert relerr(got, np.linalg.cholesky(A)) <= 1e-12


@pytest.mark.parametrize("tile,bad_tile", [(128, 1), (128, 5), (128, 8), (256, 2), (256, 6)])
def test_multistep_tail_failure_positions(cluster_factory, tile, bad_tile):
    """Failures inside the multi-step tail launch (every step chain-bound at
    these sizes): the first, a middle and the last diagonal tile.  The
    launch stops at the failing factorization (no hang), reports the block,
    leaves no factor, and the next factorization on the cluster is right."""
    from paper_1305_4886_b200 import distla
    from paper_1305_4886_b200.errors import NotPositiveDefinite
    n = tile * 9 - 11
    A = spd_matrix(n, seed=bad_tile)
    bad = min(bad_tile * tile + 17, n - 1)
    A[bad, bad] = -1.0
    cl = cluster_factory(tile=tile)
    lay = distla.make_layout(n, cl.grid, h=5)
    C = distla.distribute(cl, "C", A, "triangular", lay)
    with pytest.raises(NotPositiveDefinite) as info:
        distla.distributed_cholesky(cl, C, "L")
    assert info.value.block_index == bad // lay.block_size + 1
    assert "L" not in set(cl.remote_ls())
    A2 = _cov(n, seed=bad_tile)
    C2 = distla.distribute(cl, "C2", A2, "triangular", lay)
    L2, _ = distla.distributed_cholesky(cl, C2, "L2")
    assert relerr(distla.collect(cl, L2), np.linalg.cholesky(A2)) <= 1e-12


def test_one_launch_per_step_fallback_matches(tmp_path):
    """BGP_MULTI_STEP=0 (one launch per step in the chain-bound tail, read
    once per process) gives the same factor as the default multi-step
    launch, both against LAPACK."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from conftest import spd_matrix\n"
        "from paper_1305_4886_b200 import distla, spawn\n"
        "cl = spawn(1, tile=128); n = 128 * 12 - 5; A = spd_matrix(n, seed=2)\n"
        "C = distla.distribute(cl, 'C', A, 'triangular', distla.make_layout(n, cl.grid, h=3))\n"
        "L, _ = distla.distributed_cholesky(cl, C, 'L'); np.save(sys.argv[1], distla.collect(cl, L))\n"
        "cl.shutdown()\n") % (root, os.path.join(root, "tests"))
    out = {}
    for m in ("0", "1"):
        f = str(tmp_path / f"L{m}.npy")
        env = dict(os.environ, BGP_MULTI_STEP=m)
        subprocess.run([sys.executable, "-c", code, f], check=True, env=env, timeout=600)
        out[m] = np.load(f)
    n = out["0"].shape[0]
    want = np.linalg.cholesky(spd_matrix(n, seed=2))
    assert relerr(out["0"], want) <= 1e-12 and relerr(out["1"], want) <= 1e-12
    assert relerr(out["0"], out["1"]) <= 1e-13


@pytest.mark.parametrize("tile,ntiles,depth", [(128, 56, 2), (128, 60, 5), (256, 33, 3)])
def test_step_groups_forced_match_lapack(tmp_path, tile, ntiles, depth):
    """Step groups (the group's last launch applies `depth` panels at once,
    depth*b-deep blocks; by default groups of 5 from 64 trailing tiles at
    tile 512) forced with BGP_PAIR_STEPS=2 (read once per process, so in a
    subprocess): groups then run wherever their last step is not
    chain-bound (more than 48 / 26 trailing tiles at 128 / 256).  The
    factor and the log-determinant against LAPACK."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = tile * ntiles - 29
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from conftest import spd_matrix\n"
        "from paper_1305_4886_b200 import distla, spawn\n"
        "cl = spawn(1, tile=%d); n = %d; A = spd_matrix(n, seed=n)\n"
        "C = distla.distribute(cl, 'C', A, 'triangular', distla.make_layout(n, cl.grid, h=3))\n"
        "L, _ = distla.distributed_cholesky(cl, C, 'L')\n"
        "np.save(sys.argv[1], distla.collect(cl, L)); np.save(sys.argv[2], distla.log_det_from_chol(cl, L))\n"
        "cl.shutdown()\n") % (root, os.path.join(root, "tests"), tile, n)
    fL, fd = str(tmp_path / "L.npy"), str(tmp_path / "d.npy")
    env = dict(os.environ, BGP_PAIR_STEPS="2", BGP_GROUP_DEPTH=str(depth))
    subprocess.run([sys.executable, "-c", code, fL, fd], check=True, env=env, timeout=900)
    A = spd_matrix(n, seed=n)
    want = np.linalg.cholesky(A)
    assert relerr(np.load(fL), want) <= 1e-12
    ld = float(np.load(fd))
    assert abs(ld - np.linalg.slogdet(A)[1]) <= 1e-10 * abs(np.linalg.slogdet(A)[1])


@pytest.mark.parametrize("depth", [2, 5])
def test_step_groups_forced_failure(tmp_path, depth):
    """A non-positive pivot on a diagonal tile factored inside a step group
    (tile 3 of 56 at tile 128, groups forced): NotPositiveDefinite with the
    right block, no hang, no factor left behind."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from conftest import spd_matrix\n"
        "from paper_1305_4886_b200 import distla, spawn\n"
        "from paper_1305_4886_b200.errors import NotPositiveDefinite\n"
        "cl = spawn(1, tile=128); n = 128 * 56 - 5; A = spd_matrix(n, seed=5); bad = 3 * 128 + 40\n"
        "A[bad, bad] = -1.0; lay = distla.make_layout(n, cl.grid, h=8)\n"
        "C = distla.distribute(cl, 'C', A, 'triangular', lay)\n"
        "try:\n"
        "    distla.distributed_cholesky(cl, C, 'L'); print('NO-FAILURE')\n"
        "except NotPositiveDefinite as e:\n"
        "    ok = e.block_index == bad // lay.block_size + 1 and 'L' not in set(cl.remote_ls())\n"
        "    print('OK' if ok else 'WRONG %%d' %% e.block_index)\n"
        "cl.shutdown()\n") % (root, os.path.join(root, "tests"))
    env = dict(os.environ, BGP_PAIR_STEPS="2", BGP_GROUP_DEPTH=str(depth))
    out = subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=900, capture_output=True,
                         text=True).stdout
    assert out.strip().splitlines()[-1] == "OK", out
