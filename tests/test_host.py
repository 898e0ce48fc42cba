"""Host-side logic of the drop-in API (no GPU)."""

import math

import numpy as np
import pytest

import paper_1305_4886_b200 as bgp
from paper_1305_4886_b200 import distla, registry
from paper_1305_4886_b200.errors import (BackendUnavailable, DimensionMismatch,
                                         NotPositiveDefinite, UnknownFunction, WorkerFailure)
from paper_1305_4886_b200.grid import BlockLayout, DeviceGrid, default_h


def test_block_layout_semantics():
    lay = BlockLayout(257, 2, 3)      # the reference's padding case
    assert lay.B == 6 and lay.block_size == 43 and lay.padded_n == 258
    assert lay.block_range(2) == (44, 86)
    with pytest.raises(DimensionMismatch):
        BlockLayout(0, 1, 1)


@pytest.mark.parametrize("n,D", [(1, 1), (999, 1), (1000, 1), (1001, 1), (67275, 1),
                                 (67275, 3), (5000, 4), (131072, 1)])
def test_default_h_is_smallest(n, D):
    h = default_h(n, D)
    assert math.ceil(n / (h * D)) <= 1000
    assert h == 1 or math.ceil(n / ((h - 1) * D)) > 1000


@pytest.mark.parametrize("G,shape", [(1, (1, 1)), (2, (1, 2)), (4, (2, 2)), (8, (2, 4))])
def test_device_grid_shapes_and_partition(G, shape):
    g = DeviceGrid(G)
    assert g.shape == shape and g.P == G
    T = 11
    owned = [g.owned_tiles(r, T) for r in range(G)]
    flat = sorted(t for o in owned for t in o)
    assert flat == sorted((I, J) for J in range(T) for I in range(J, T))
    # 2-D block-cyclic: every tile of a tile column lives in one process column
    pr, pc = shape
    for I, J in flat:
        assert g.owner(I, J) // pr == J % pc
    for r in range(1, G + 1):
        assert g.coord_to_rank(*g.rank_to_coord(r)) == r


def test_registry_has_every_builtin_generator():
    for kern in bgp.gp.BUILTIN_KERNELS:
        for part in ("cov", "cross", "pred", "predvar"):
            assert isinstance(registry.device_generator(f"gen.{kern}.{part}"),
                              registry.DeviceGenerator)
    g = registry.device_generator("gen.matern-nugget.cov")
    assert g.nugget and not registry.device_generator("gen.matern-nugget.cross").nugget
    assert registry.device_generator("gen.sqexp-nugget.cov").nugget
    with pytest.raises(UnknownFunction):
        registry.device_generator("gen.cubic.cov")
    registry.register("gen.host_callable", lambda p, inp, i, j: i * 0.0)
    with pytest.raises(UnknownFunction):
        registry.device_generator("gen.host_callable")


def test_builtin_kernel_table():
    assert bgp.gp.BUILTIN_KERNELS == {"sqexp": 2, "matern": 2, "matern-nugget": 3,
                                      "matern-product-nugget": 4, "white": 1}
    with pytest.raises(DimensionMismatch):
        bgp.gp.builtin_spec("cubic", [0.0])


def test_matern_host_utilities():
    from paper_1305_4886_b200.gp import matern_correlation, sqexp_correlation
    from scipy.special import gamma, kv
    for nu in (1.5, 2.5):
        d = np.linspace(0.05, 6.0, 10)
        s = np.sqrt(2 * nu) * d / 1.7
        want = (2 ** (1 - nu) / gamma(nu)) * s ** nu * kv(nu, s)
        np.testing.assert_allclose(matern_correlation(d, 1.7, nu), want, rtol=1e-10)
    assert matern_correlation(0.0, 2.0, 0.5) == 1.0
    assert abs(sqexp_correlation(2.0, 2.0) - np.exp(-0.5)) < 1e-15
    with pytest.raises(ValueError):
        matern_correlation(1.0, 0.0, 0.5)


def test_api_surface_matches_reference_names():
    for name in ("collect", "collect_diagonal", "construct_distributed",
                 "construct_rnorm_distributed", "crossprod_mat_vec", "crossprod_self",
                 "crossprod_self_diag", "distribute", "distributed_cholesky",
                 "log_det_from_chol", "make_layout", "mult_chol", "sum_squares",
                 "triangular_solve"):
        assert callable(getattr(distla, name))
    for name in ("KrigeProblem", "CovarianceSpec", "builtin_spec", "OptResult"):
        assert hasattr(bgp.gp, name)
    assert bgp.spawn is bgp.transport.spawn


def test_spawn_rejects_cpu_backends():
    with pytest.raises(BackendUnavailable):
        bgp.spawn(1, backend="in-process")


def test_spawn_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(BackendUnavailable):
        bgp.spawn(1)


def test_exceptions_pickle():
    import pickle
    for exc in (NotPositiveDefinite(3, "x"), WorkerFailure(2, RuntimeError("boom"))):
        back = pickle.loads(pickle.dumps(exc))
        assert type(back) is type(exc) and str(back) == str(exc)
