"""The CPU oracle pinned against the reference's own outputs (no GPU).

The oracle (oracle/blockgp_oracle.py) is the checker for the CUDA path; it
is trusted only because these tests reproduce, from the oracle, every
fixture that tests/golden/make_golden.py obtained by running the reference
`blockgp` package, plus the survey's scalar goldens for BASELINE configs
1 and 4.
"""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, relerr
from oracle import blockgp_oracle as orc


@pytest.mark.parametrize("key", ["matern05", "matern15", "matern25", "maternnn", "sqexp",
                                 "sqexpnug", "white", "product"])
def test_generators_match_reference(golden, golden_scalars, key):
    meta = golden_scalars[f"con_{key}"]
    X, Xp = golden["con_X"], golden["con_Xp"]
    inputs = {"coords": X, "pred_coords": Xp}
    inputs.update(meta["inputs"])
    kern, theta = meta["kernel"], np.array(meta["theta"])
    bs = math.ceil(37 / 2)
    C = orc.construct_triangular(orc.Generator(f"gen.{kern}.cov"), theta, inputs, 37, bs)
    np.testing.assert_array_equal(C[:37, :37], golden[f"con_{key}_cov"])
    Cx = orc.construct_rectangular(orc.Generator(f"gen.{kern}.cross"), theta, inputs, 37, 11, bs, 11)
    np.testing.assert_array_equal(Cx[:37, :11], golden[f"con_{key}_cross"])
    Cp = orc.construct_triangular(orc.Generator(f"gen.{kern}.pred"), theta, inputs, 11, 11)
    np.testing.assert_array_equal(Cp[:11, :11], golden[f"con_{key}_pred"])
    pv = orc.construct_vector(orc.Generator(f"gen.{kern}.predvar"), theta, inputs, 11, 11)
    np.testing.assert_array_equal(pv[:11], golden[f"con_{key}_predvar"])


@pytest.mark.parametrize("n", [37, 257, 300])
def test_linear_algebra_matches_reference(golden, golden_scalars, n):
    k = f"la{n}"
    sc = golden_scalars[k]
    bs = sc["block"]
    A = orc.pad_triangular(golden[f"{k}_A"], n, bs)
    L = orc.cholesky(A, bs)
    assert relerr(L[:n, :n], golden[f"{k}_L"]) <= 1e-14
    pn = L.shape[0]
    b = np.zeros(pn)
    b[:n] = golden[f"{k}_b"]
    u = orc.solve_vector(L, b, bs, forward=True)
    x = orc.solve_vector(L, u, bs, forward=False)
    assert relerr(u[:n], golden[f"{k}_u"]) <= 1e-14
    assert relerr(x[:n], golden[f"{k}_x"]) <= 1e-13
    R = np.zeros((pn, 7))
    R[:n] = golden[f"{k}_R"]
    W = orc.solve_rect(L, R, bs, forward=True)
    Wb = orc.solve_rect(L, R, bs, forward=False)
    assert relerr(W[:n], golden[f"{k}_W"]) <= 1e-14
    assert relerr(Wb[:n], golden[f"{k}_Wb"]) <= 1e-13
    assert relerr(orc.xprod_mat_vec(W, u, n, 7), golden[f"{k}_w"]) <= 1e-14
    assert relerr(orc.xprod_self(W, n, 7), golden[f"{k}_S"]) <= 1e-14
    assert relerr(orc.xprod_self_diag(W, n, 7), golden[f"{k}_d"]) <= 1e-14
    assert abs(orc.logdet(L, n, bs) - sc["logdet"]) <= 1e-14 * abs(sc["logdet"])
    assert abs(orc.sumsq(u, n, bs) - sc["ssq"]) <= 1e-14 * abs(sc["ssq"])


def test_not_pd_block_index(golden, golden_scalars):
    A = orc.pad_triangular(-np.eye(6), 6, 6)
    with pytest.raises(orc.OracleNotPD) as e:
        orc.cholesky(A, 6)
    assert e.value.block_index == golden_scalars["npd_minus_identity_block"] == 1
    A = orc.pad_triangular(golden["npd_A"], 40, 20)
    with pytest.raises(orc.OracleNotPD) as e:
        orc.cholesky(A, 20)
    assert e.value.block_index == golden_scalars["npd_A_block_h2"]


def test_singular_diagonal_detected(golden_scalars):
    L = np.array([[1.0, 0.0], [1.0, 0.0]])
    with pytest.raises(orc.OracleSingular):
        orc.solve_vector(L, np.ones(2), 2)
    assert golden_scalars["singular_detected"]


@pytest.mark.parametrize("key", ["gp400", "gp300m15", "gp250m25", "gp300sq"])
def test_gp_end_to_end_matches_reference(golden, golden_scalars, key):
    sc = golden_scalars[key]
    prob = orc.OracleProblem(sc["kernel"], golden[f"{key}_X"], golden[f"{key}_y"],
                             sc["theta"], pred_coords=golden[f"{key}_Xp"], **sc["inputs"])
    ll = prob.log_density()
    assert abs(ll - sc["ll"]) <= 1e-13 * abs(sc["ll"])
    mean, se = prob.predict(se_fit=True)
    assert relerr(mean, golden[f"{key}_mean"]) <= 1e-12
    assert relerr(se, golden[f"{key}_se"]) <= 1e-12
    assert relerr(prob.prediction_variance(), golden[f"{key}_PV"]) <= 1e-12


def test_config1_recipe_and_loglik(golden, golden_scalars):
    """The 8d input recipe reproduces the survey's C1 ll (pins the inputs)."""
    kern, X, theta, extra, z = orc.config_inputs(1)
    y = np.linalg.cholesky(orc.dense_cov(kern, theta, X, **extra)) @ z
    assert relerr(y, golden["c1_y"]) <= 1e-13
    prob = orc.OracleProblem(kern, X, golden["c1_y"], theta, **extra)
    ll = prob.log_density()
    assert abs(ll - golden_scalars["c1"]["ll"]) <= 1e-12 * abs(ll)
    assert abs(ll - golden_scalars["c1"]["survey_ll"]) <= 1e-12 * abs(ll)


def test_config4_inputs_consistent_with_survey(c4_scalars):
    """Frozen C4 inputs (make_c4_inputs.py) reproduce BASELINE.md 3's scalars."""
    s = c4_scalars["survey"]
    assert abs(c4_scalars["logdet"] - s["logdet"]) <= 1e-12 * abs(s["logdet"])
    assert c4_scalars["ssq_z"] == pytest.approx(s["ssq"], rel=1e-14)
    assert c4_scalars["norm_y"] == pytest.approx(s["norm_y"], rel=1e-12)
    assert abs(c4_scalars["ll_from_this_factor"] - s["ll"]) <= 1e-10 * abs(s["ll"])
    # the survey's ||L||_F includes the reference's 45 identity-padded rows
    # (block 990: padded_n = 67,320)
    assert math.hypot(c4_scalars["norm_L_fro"], math.sqrt(67320 - 67275)) == \
        pytest.approx(s["norm_L_fro"], rel=1e-12)


def test_config4_input_recipe():
    kern, X, theta, extra, z = orc.config_inputs(4)
    assert X.shape == (67275, 2) and kern == "matern-nugget"
    data = np.load("tests/golden/c4_inputs.npz")
    np.testing.assert_array_equal(data["X"], X)
    np.testing.assert_array_equal(data["z"], z)


def test_full_eval_packed_sweep_matches_reference(golden, golden_scalars):
    """oracle/full_eval.py (the packed-block restatement timed on the GPU
    host as the full CPU baseline) reproduces the reference's C1 ll."""
    from oracle import full_eval
    kern, X, theta, extra, z = orc.config_inputs(1)
    r = full_eval.log_density(X, golden["c1_y"], theta)
    assert r["block"] == 683
    assert abs(r["ll"] - golden_scalars["c1"]["ll"]) <= 1e-13 * abs(r["ll"])


def test_full_size_reference_fixtures_agree_with_survey():
    """The full-size fixtures (make_full_configs.py, produced by the
    reference) reproduce BASELINE.md 3's survey goldens: C2's ten ll to the
    survey's 12 significant digits, C3's ll and ||mean||, ||se||, and the
    coordinates regenerate from the seed."""
    import json
    meta = json.load(open(os.path.join(GOLDEN, "full_configs.json")))
    c2 = [-7686.62544235, -4553.77461647, -4574.36131115, -5658.81011183, -7290.93691243,
          -9256.45042656, -11437.3571029, -13759.4716896, -16173.2526993, -18644.7801649]
    for got, want in zip(meta["c2"]["ll"], c2):
        assert abs(got - want) <= 5e-12 * abs(want)
    c3 = meta["c3"]
    assert abs(c3["ll"] - (-1206.4571584386722)) <= 1e-10 * 1206.46
    assert c3["norm_mean"] == pytest.approx(61.725485129258466, rel=1e-12)
    assert c3["norm_se"] == pytest.approx(12.093826573490732, rel=1e-12)
    for cfg, n in ((2, None), (3, None), (5, 16384), (4, None)):
        X = orc.config_inputs(cfg, n=n)[1]
        key = {2: "c2", 3: "c3", 5: "c5s", 4: "c4_lead"}[cfg]
        assert float(np.sum(X)) == meta[key]["X"]["sum"]


def test_sub_evaluation_sampler_extrapolates_by_op_counts():
    from oracle.cpu_baseline import SubEvalSampler, op_counts
    kern, X, theta, extra, z = orc.config_inputs(1)
    s = SubEvalSampler(X, theta, blocks=2)
    assert s.n_sub == 2 * s.bs and s.counts == op_counts(len(X), s.bs)
    t, wall = s.sample()
    assert set(t) == {"construct", "potrf", "trsm", "syrk", "gemv", "trsv"}  # no GEMM in 2 blocks
    t["gemm"] = t["syrk"]
    total, chol = s.extrapolate(t)
    assert 0 < chol < total and wall > 0
