"""CUDA path against fixtures produced by the reference itself.

tests/golden/golden_small.npz + golden_scalars.json come from
tests/golden/make_golden.py (the reference `blockgp` run in the build
container).  Tolerances: 1e-14 absolute on covariance entries
(pkg/tests/test_distla.py:50), normwise 1e-9 on L / predictions and 1e-10
relative on log-likelihoods (BASELINE.json north star).
"""

import numpy as np
import pytest

from conftest import relerr

pytestmark = pytest.mark.gpu

GEN_CASES = ["matern05", "matern15", "matern25", "maternnn", "sqexp", "sqexpnug",
             "white", "product"]


@pytest.mark.parametrize("key", GEN_CASES)
@pytest.mark.parametrize("tile", [128, 256])
def test_construct_every_generator(cluster_factory, golden, golden_scalars, key, tile):
    from paper_1305_4886_b200 import distla
    meta = golden_scalars[f"con_{key}"]
    cl = cluster_factory(tile=tile)
    X, Xp = golden["con_X"], golden["con_Xp"]
    inputs = {"coords": X, "pred_coords": Xp}
    inputs.update(meta["inputs"])
    cl.push("inp", inputs)
    rows = distla.make_layout(37, cl.grid, h=2)
    cols = distla.make_layout(11, cl.grid, h=1)
    kern, theta = meta["kernel"], meta["theta"]
    t = distla.construct_distributed(cl, "C", "triangular", f"gen.{kern}.cov", theta,
                                     inputs_name="inp", row_layout=rows)
    np.testing.assert_allclose(distla.collect(cl, t), golden[f"con_{key}_cov"], rtol=0, atol=1e-14)
    r = distla.construct_distributed(cl, "Cx", "rectangular", f"gen.{kern}.cross", theta,
                                     inputs_name="inp", row_layout=rows, col_layout=cols)
    np.testing.assert_allclose(distla.collect(cl, r), golden[f"con_{key}_cross"], rtol=0, atol=1e-14)
    p = distla.construct_distributed(cl, "Cp", "triangular", f"gen.{kern}.pred", theta,
                                     inputs_name="inp", row_layout=cols)
    np.testing.assert_allclose(distla.collect(cl, p), golden[f"con_{key}_pred"], rtol=0, atol=1e-14)
    v = distla.construct_distributed(cl, "pv", "vector", f"gen.{kern}.predvar", theta,
                                     inputs_name="inp", row_layout=cols)
    np.testing.assert_array_equal(distla.collect(cl, v), golden[f"con_{key}_predvar"])


@pytest.mark.parametrize("n", [37, 257, 300])
@pytest.mark.parametrize("tile", [128, 256])
def test_linear_algebra_vs_reference(cluster_factory, golden, golden_scalars, n, tile):
    from paper_1305_4886_b200 import distla
    k = f"la{n}"
    sc = golden_scalars[k]
    cl = cluster_factory(tile=tile)
    lay = distla.make_layout(n, cl.grid, h=sc["h"])
    lc = distla.make_layout(7, cl.grid, h=1)
    C = distla.distribute(cl, "C", golden[f"{k}_A"], "triangular", lay)
    L, _ = distla.distributed_cholesky(cl, C, "L")
    assert relerr(distla.collect(cl, L), golden[f"{k}_L"]) <= 1e-12
    bd = distla.distribute(cl, "b", golden[f"{k}_b"], "vector", lay)
    u = distla.triangular_solve(cl, L, bd, "u", side="forward")
    x = distla.triangular_solve(cl, L, u, "x", side="back")
    assert relerr(distla.collect(cl, u), golden[f"{k}_u"]) <= 1e-12
    assert relerr(distla.collect(cl, x), golden[f"{k}_x"]) <= 1e-12
    Rd = distla.distribute(cl, "R", golden[f"{k}_R"], "rectangular", lay, lc)
    W = distla.triangular_solve(cl, L, Rd, "W", side="forward")
    Wb = distla.triangular_solve(cl, L, Rd, "Wb", side="back")
    assert relerr(distla.collect(cl, W), golden[f"{k}_W"]) <= 1e-12
    assert relerr(distla.collect(cl, Wb), golden[f"{k}_Wb"]) <= 1e-12
    assert relerr(distla.collect(cl, distla.crossprod_mat_vec(cl, W, u, "w")), golden[f"{k}_w"]) <= 1e-12
    assert relerr(distla.collect(cl, distla.crossprod_self(cl, W, "S")), golden[f"{k}_S"]) <= 1e-12
    assert relerr(distla.collect(cl, distla.crossprod_self_diag(cl, W, "d")), golden[f"{k}_d"]) <= 1e-12
    assert abs(distla.log_det_from_chol(cl, L) - sc["logdet"]) <= 1e-12 * abs(sc["logdet"])
    assert abs(distla.sum_squares(cl, u) - sc["ssq"]) <= 1e-12 * abs(sc["ssq"])


def _spec(kern, X, Xp, extra):
    from paper_1305_4886_b200.gp import CovarianceSpec, builtin_spec
    if kern == "sqexp-nugget":
        ids = {p: f"gen.sqexp-nugget.{p}" for p in ("cov", "cross", "pred", "predvar")}
        return CovarianceSpec(cov_fn=ids["cov"], cross_cov_fn=ids["cross"], pred_cov_fn=ids["pred"],
                              pred_var_fn=ids["predvar"],
                              inputs={"coords": X, "pred_coords": Xp}, n_params=3)
    return builtin_spec(kern, X, Xp, **extra)


@pytest.mark.parametrize("key", ["gp400", "gp300m15", "gp250m25", "gp300sq"])
@pytest.mark.parametrize("tile", [128, 256])
def test_krige_problem_vs_reference(cluster_factory, golden, golden_scalars, key, tile):
    from paper_1305_4886_b200.gp import KrigeProblem
    sc = golden_scalars[key]
    X, Xp, y = golden[f"{key}_X"], golden[f"{key}_Xp"], golden[f"{key}_y"]
    cl = cluster_factory(tile=tile)
    prob = KrigeProblem(cl, "g", _spec(sc["kernel"], X, Xp, sc["inputs"]), y,
                        np.array(sc["theta"]), m=len(Xp))
    ll = prob.log_density()
    assert abs(ll - sc["ll"]) <= 1e-10 * abs(sc["ll"])
    assert abs(ll - sc["ll_P3h2"]) <= 1e-10 * abs(sc["ll"])
    mean, se = prob.predict(se_fit=True)
    assert relerr(mean, golden[f"{key}_mean"]) <= 1e-9
    assert relerr(se, golden[f"{key}_se"]) <= 1e-9
    PV = prob.prediction_variance()
    assert relerr(PV, golden[f"{key}_PV"]) <= 1e-9
    assert relerr(np.diag(PV), se ** 2) <= 1e-12


@pytest.mark.parametrize("tile", [128, 256, 512])
def test_config1_loglik(cluster_factory, golden, golden_scalars, tile):
    """BASELINE config 1 at full size (n = 2048) against the reference ll."""
    from oracle.blockgp_oracle import config_inputs
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    kern, X, theta, extra, _ = config_inputs(1)
    cl = cluster_factory(tile=tile)
    prob = KrigeProblem(cl, "c1", builtin_spec(kern, X, **extra), golden["c1_y"], theta)
    ll = prob.log_density()
    want = golden_scalars["c1"]["ll"]
    assert abs(ll - want) <= 1e-10 * abs(want)
    assert abs(ll - golden_scalars["c1"]["survey_ll"]) <= 1e-10 * abs(want)
    from paper_1305_4886_b200 import distla
    assert relerr(distla.collect(cl, prob._handles["u"]), golden["c1_u"]) <= 1e-9


def test_config2_theta_sweep_n2048(cluster_factory, golden, golden_scalars):
    """BASELINE config 2's 10-range sweep at n = 2048 (same recipe)."""
    from oracle.blockgp_oracle import config_inputs
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    kern, X, theta, extra, _ = config_inputs(2, n=2048)
    cl = cluster_factory(tile=256)
    prob = KrigeProblem(cl, "c2", builtin_spec(kern, X, **extra), golden["c2s_y"], theta)
    for rho, want in zip(np.linspace(0.02, 0.2, 10), golden_scalars["c2_n2048"]["ll"]):
        ll = prob.log_density(np.array([2.0, rho, 0.05]))
        assert abs(ll - want) <= 1e-10 * abs(want)


def test_freshness_no_device_work(cluster_factory, golden, golden_scalars):
    from paper_1305_4886_b200.gp import KrigeProblem
    sc = golden_scalars["gp400"]
    cl = cluster_factory(tile=128)
    prob = KrigeProblem(cl, "g", _spec(sc["kernel"], golden["gp400_X"], golden["gp400_Xp"],
                                       sc["inputs"]), golden["gp400_y"], np.array(sc["theta"]))
    first = prob.log_density()
    before, launches = cl.stats["collectives"], cl.launches()
    assert prob.log_density() == first
    assert cl.stats["collectives"] == before and cl.launches() == launches
    b = prob.log_density(np.array(sc["theta"]) * 1.1)
    assert b != first and cl.launches() > launches
