"""Simulation on the GPU: rank streams and conditional / unconditional draws.

The reference's P = 1 draws (tests/golden: RankStream(21, 1) and
KrigeProblem.simulate_realizations with seed 21) are reproduced here from the
same Philox4x64-10 stream, so the realizations must agree to rounding
(bg/rng.py:18-28, bg/gp/problem.py:267-300; pkg/tests/test_gp.py TestSimulate).
"""

import numpy as np
import pytest

from conftest import exp_cov, relerr

pytestmark = pytest.mark.gpu


def test_rank_stream_matches_reference(cluster_factory, golden):
    from paper_1305_4886_b200 import distla
    cl = cluster_factory(seed=21, tile=128)
    lay = distla.make_layout(1000, cl.grid, h=1)
    z = distla.construct_rnorm_distributed(cl, "z", "vector", lay)
    np.testing.assert_allclose(distla.collect(cl, z), golden["rng_seed21_rank1"], rtol=0, atol=1e-13)


def test_simulations_match_reference_draws(cluster_factory, golden, golden_scalars):
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    sc = golden_scalars["sim"]
    cl = cluster_factory(seed=sc["seed"], tile=128)
    spec = builtin_spec("matern-nugget", golden["sim_X"], golden["sim_Xp"], nu=sc["nu"])
    prob = KrigeProblem(cl, "s", spec, golden["sim_y"], np.array(sc["theta"]), m=9)
    assert relerr(prob.simulate_realizations(4, post=False), golden["sim_unc"]) <= 1e-12
    assert relerr(prob.simulate_realizations(3, post=True), golden["sim_post"]) <= 1e-9
    assert relerr(prob.simulate_realizations(2, post=False), golden["sim_unc2"]) <= 1e-12


def _prob(cl, m=5):
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    rng = np.random.default_rng(14)
    coords = np.sort(rng.uniform(0, 10, 20))
    pred = np.linspace(1, 9, m)
    theta = np.array([1.5, 2.0, 0.1])
    y = np.linalg.cholesky(exp_cov(coords, *theta)) @ rng.standard_normal(20)
    return KrigeProblem(cl, "t", builtin_spec("matern-nugget", coords, pred), y, theta, m=m)


def test_zero_noise_unconditional_is_mean(cluster_factory):
    cl = cluster_factory(tile=128)
    sims = _prob(cl).simulate_realizations(3, post=False, zero_noise=True)
    np.testing.assert_allclose(sims, np.zeros((20, 3)), atol=1e-12)


def test_zero_noise_conditional_is_prediction(cluster_factory):
    cl = cluster_factory(tile=128)
    prob = _prob(cl)
    mean = prob.predict()
    sims = prob.simulate_realizations(2, post=True, zero_noise=True)
    np.testing.assert_allclose(sims, np.broadcast_to(mean[:, None], sims.shape), atol=1e-10)


def test_deterministic_given_seed_and_shapes(cluster_factory):
    out = []
    for _ in range(2):
        cl = cluster_factory(seed=21, tile=128)
        out.append(_prob(cl).simulate_realizations(4, post=True).tobytes())
    assert out[0] == out[1]
    cl = cluster_factory(tile=128)
    prob = _prob(cl)
    assert prob.simulate_realizations(7, post=False).shape == (20, 7)
    assert prob.simulate_realizations(7, post=True).shape == (5, 7)


@pytest.mark.parametrize("tile,n,m", [(128, 300, 140), (256, 700, 300)])
def test_mult_rect_vs_numpy(cluster_factory, tile, n, m):
    from paper_1305_4886_b200 import distla
    cl = cluster_factory(tile=tile)
    rng = np.random.default_rng(10)
    Ls = np.tril(rng.standard_normal((n, n)))
    Z = rng.standard_normal((n, m))
    rows, cols = distla.make_layout(n, cl.grid, h=1), distla.make_layout(m, cl.grid, h=1)
    L = distla.distribute(cl, "L", Ls, "triangular", rows)
    Zd = distla.distribute(cl, "Z", Z, "rectangular", rows, cols)
    assert relerr(distla.collect(cl, distla.mult_chol(cl, L, Zd, "Y")), Ls @ Z) <= 1e-12


def test_rnorm_moments(cluster_factory):
    from paper_1305_4886_b200 import distla
    cl = cluster_factory(seed=3, tile=128)
    rows, cols = distla.make_layout(1000, cl.grid, h=2), distla.make_layout(100, cl.grid, h=1)
    Z = distla.collect(cl, distla.construct_rnorm_distributed(cl, "Z", "rectangular", rows, cols))
    assert abs(Z.mean()) < 0.01 and abs(Z.var() - 1.0) < 0.02 and np.all(np.isfinite(Z))
