"""The C ABI (include/bgp.h) driven directly through ctypes, the way a
reference-side binding would call it: pack a dense SPD
matrix into tiles, factor (bgp_potrf), forward/back solve (bgp_trsv),
log-determinant and sum of squares, unpack -- compared with LAPACK / numpy.
No package-level Python sits between the test and the library."""

import ctypes

import numpy as np
import pytest

from conftest import relerr, spd_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture
def abi():
    import torch

    from paper_1305_4886_b200 import _lib
    lib = _lib.load()
    ctx = ctypes.c_void_p()
    assert lib.bgp_init(0, ctypes.byref(ctx)) == 0
    stream = torch.cuda.current_stream().cuda_stream
    yield lib, ctx, stream, torch
    torch.cuda.synchronize()
    lib.bgp_finalize(ctx)


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


@pytest.mark.parametrize("n,tile", [(300, 128), (1000, 256), (1500, 512), (2048, 256)])
def test_potrf_trsv_logdet_through_the_abi(abi, n, tile):
    lib, ctx, s, torch = abi
    A = spd_matrix(n, seed=n)
    T = -(-n // tile)
    dense = torch.from_numpy(A).cuda()
    tiles = torch.empty((T * (T + 1) // 2, tile, tile), dtype=torch.float64, device="cuda")
    assert lib.bgp_pack(ctx, 0, _p(dense), n, n, n, tile, _p(tiles), s) == 0  # BGP_TRI
    info = ctypes.c_int64(-1)
    assert lib.bgp_potrf(ctx, _p(tiles), n, tile, ctypes.byref(info), s) == 0
    assert info.value == 0
    out = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    assert lib.bgp_unpack(ctx, 0, _p(tiles), n, n, tile, _p(out), n, s) == 0
    L = np.linalg.cholesky(A)
    assert relerr(out.cpu().numpy(), L) <= 1e-12

    rhs = np.random.default_rng(n).standard_normal(n)
    x = torch.zeros(T * tile, dtype=torch.float64, device="cuda")
    x[:n] = torch.from_numpy(rhs).cuda()
    assert lib.bgp_trsv(ctx, _p(tiles), n, tile, _p(x), 0, ctypes.byref(info), s) == 0 and info.value == 0
    u = x[:n].cpu().numpy()
    assert relerr(u, np.linalg.solve(L, rhs)) <= 1e-12
    ssq = ctypes.c_double()
    assert lib.bgp_sumsq(ctx, _p(x), n, ctypes.byref(ssq), s) == 0
    assert abs(ssq.value - u @ u) <= 1e-12 * (u @ u)
    assert lib.bgp_trsv(ctx, _p(tiles), n, tile, _p(x), 1, ctypes.byref(info), s) == 0 and info.value == 0
    assert relerr(x[:n].cpu().numpy(), np.linalg.solve(A, rhs)) <= 1e-10

    ld = ctypes.c_double()
    assert lib.bgp_logdet(ctx, _p(tiles), n, tile, ctypes.byref(ld), ctypes.byref(info), s) == 0
    assert info.value == 0
    want = np.linalg.slogdet(A)[1]
    assert abs(ld.value - want) <= 1e-12 * abs(want)


def test_potrf_reports_first_bad_pivot_row(abi):
    lib, ctx, s, torch = abi
    n, tile = 700, 128
    A = spd_matrix(n, seed=3)
    A[517, 517] = -5.0
    T = -(-n // tile)
    dense = torch.from_numpy(A).cuda()
    tiles = torch.empty((T * (T + 1) // 2, tile, tile), dtype=torch.float64, device="cuda")
    assert lib.bgp_pack(ctx, 0, _p(dense), n, n, n, tile, _p(tiles), s) == 0
    info = ctypes.c_int64(0)
    assert lib.bgp_potrf(ctx, _p(tiles), n, tile, ctypes.byref(info), s) == 0
    assert info.value == 518  # 1-based row, LAPACK convention


def test_bad_arguments_are_rejected(abi):
    lib, ctx, s, torch = abi
    info = ctypes.c_int64(0)
    t = torch.zeros((1, 128, 128), dtype=torch.float64, device="cuda")
    assert lib.bgp_potrf(ctx, _p(t), 100, 100, ctypes.byref(info), s) != 0  # tile not a multiple of 128


def test_gemm_launches_on_two_streams_do_not_share_counters(abi):
    """A trailing update and a panel solve enqueued on two streams with no
    host synchronisation between them (they overlap on the GPU): each launch
    owns its task counter (a ring slot zeroed on its own stream), so neither
    re-runs nor steals the other's tasks.  Both results against numpy."""
    lib, ctx, s, torch = abi
    b, nt = 256, 60
    rng = np.random.default_rng(4)
    mats = lambda k: torch.from_numpy(rng.standard_normal((k, b, b))).cuda()  # noqa: E731
    C, A, B = mats(nt), mats(nt), mats(nt)
    C0 = C.clone()
    items = torch.tensor([[k, k, (k + 1) % nt, 0] for k in range(nt)], dtype=torch.int32).cuda()
    L = np.linalg.cholesky(spd_matrix(b, seed=1))
    Linv = torch.from_numpy(np.ascontiguousarray(np.linalg.inv(L).T)).cuda()  # column-major tile
    X = mats(40)
    X0 = X.clone()
    s2 = torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        assert lib.bgp_tile_update(ctx, _p(C), _p(A), _p(B), _p(items), nt, b, s) == 0
        assert lib.bgp_panel_trsm_inv(ctx, _p(Linv), _p(X), 40, b, s2.cuda_stream) == 0
        assert lib.bgp_panel_trsm_inv(ctx, _p(Linv), _p(X), 40, b, s2.cuda_stream) == 0
    torch.cuda.synchronize()
    m = lambda t: t.cpu().numpy().transpose(0, 2, 1)  # noqa: E731  column-major tiles -> matrices
    a, bb, c0 = m(A), m(B), m(C0)
    want = np.stack([c0[k] - 3 * a[k] @ bb[(k + 1) % nt].T for k in range(nt)])
    assert relerr(m(C), want) <= 1e-12
    Li = np.linalg.inv(L)
    xw = m(X0)
    for _ in range(6):
        xw = xw @ Li.T
    assert relerr(m(X), xw) <= 1e-11
