"""Parity at the FULL BASELINE config sizes against the reference's outputs.

Fixtures: tests/golden/full_configs.{npz,json} (make_full_configs.py: the
reference `blockgp` run at C2 / C3 / C5-kernel sizes in the build container)
and c4_inputs.npz / c4_scalars.json (BASELINE.md 3's survey goldens).
Tolerances are the north star's: log-likelihood relative 1e-10, L and
predictions normwise 1e-9; logdet relative 1e-12.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full():
    with open(os.path.join(GOLDEN, "full_configs.json")) as f:
        meta = json.load(f)
    return meta, np.load(os.path.join(GOLDEN, "full_configs.npz"))


def _inputs(config, meta, n=None):
    from oracle.blockgp_oracle import config_inputs
    kern, X, theta, extra, _ = config_inputs(config, n=n)
    ck = meta["X"]
    assert float(np.sum(X)) == ck["sum"] and list(X.ravel()[:4]) == ck["first"], \
        "coordinate generator drifted from the frozen recipe"
    return kern, X, theta, extra


@pytest.mark.parametrize("tile", [256, 512])
def test_c2_ten_loglik_evaluations(cluster_factory, full, tile):
    """C2: n = 16,384 Matern 3/2, ll at the ten ranges (bg/gp/problem.py:170-183)."""
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    meta, arr = full
    m = meta["c2"]
    kern, X, theta, extra = _inputs(2, m)
    cl = cluster_factory(tile=tile)
    prob = KrigeProblem(cl, "c2", builtin_spec(kern, X, **extra), arr["c2_y"], theta)
    for rho, want in zip(m["rho"], m["ll"]):
        got = prob.log_density(np.array([2.0, rho, 0.05]))
        assert abs(got - want) <= 1e-10 * abs(want), (rho, got, want)


@pytest.mark.parametrize("tile", [256])
def test_c3_kriging_mean_and_se_vectors(cluster_factory, full, tile):
    """C3: n = 32,768, m = 4,096: ll, and the full mean / se vectors of
    predict(se_fit=True) normwise (bg/gp/problem.py:221-244)."""
    from oracle.blockgp_oracle import c3_pred_coords
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    meta, arr = full
    m = meta["c3"]
    kern, X, theta, extra = _inputs(3, m)
    Xp = c3_pred_coords()
    cl = cluster_factory(tile=tile)
    prob = KrigeProblem(cl, "c3", builtin_spec(kern, X, Xp, **extra), arr["c3_y"], theta, m=len(Xp))
    ll = prob.log_density()
    assert abs(ll - m["ll"]) <= 1e-10 * abs(m["ll"])
    mean, se = prob.predict(se_fit=True)
    assert relerr(mean, arr["c3_mean"]) <= 1e-9
    assert relerr(se, arr["c3_se"]) <= 1e-9


def test_c5_kernel_sqexp_nugget_at_16384(cluster_factory, full):
    """C5's kernel (squared exponential + nugget, registered through the
    reference's _make_pairwise) at n = 16,384 against the reference."""
    from paper_1305_4886_b200 import distla
    from paper_1305_4886_b200.gp import CovarianceSpec, KrigeProblem
    meta, arr = full
    m = meta["c5s"]
    _, X, theta, _ = _inputs(5, m, n=16384)
    spec = CovarianceSpec(cov_fn="gen.sqexp-nugget.cov", cross_cov_fn="gen.sqexp-nugget.cross",
                          pred_cov_fn="gen.sqexp-nugget.pred", pred_var_fn="gen.sqexp-nugget.predvar",
                          inputs={"coords": X}, n_params=3)
    cl = cluster_factory(tile=512)
    prob = KrigeProblem(cl, "c5s", spec, arr["c5s_y"], theta)
    ll = prob.log_density()
    assert abs(ll - m["ll"]) <= 1e-10 * abs(m["ll"])
    logdet = distla.log_det_from_chol(cl, prob._handles["L"])
    ssq = distla.sum_squares(cl, prob._handles["u"])
    assert abs(logdet - m["logdet"]) <= 1e-12 * abs(m["logdet"])
    assert abs(ssq - m["ssq"]) <= 1e-10 * abs(m["ssq"])


def _dense_lead(L, k):
    """Leading k x k block of a packed-tile lower factor, on the device."""
    import torch
    b = L.tile
    T = -(-L.n // b)
    kt = k // b
    out = torch.zeros((k, k), dtype=torch.float64, device=L.data.device)
    for J in range(kt):
        for I in range(J, kt):
            t = J * T - J * (J - 1) // 2 + (I - J)
            out[I * b:(I + 1) * b, J * b:(J + 1) * b] = L.data[t].T  # tiles are column-major
    return out


@pytest.mark.parametrize("tile", [256, 512])
def test_c4_full_size_factor_and_loglik(cluster_factory, full, c4_scalars, tile):
    """C4 (n = 67,275): ll and logdet against the survey's reference run,
    ||L||_F against the reference's (which counts its 45 identity-padded
    rows at block 990), the leading 4,096 rows of L against reference
    probes, and the residual ||(L L^T - C) x|| / ||C x|| at full size."""
    import ctypes

    import torch

    from paper_1305_4886_b200 import distla
    from paper_1305_4886_b200.gp import KrigeProblem, builtin_spec
    meta, arr = full
    s = c4_scalars["survey"]
    d = np.load(os.path.join(GOLDEN, "c4_inputs.npz"))
    X, y = d["X"], d["y"]
    n = len(y)
    theta = np.array([1.0, 0.08, 0.02])
    cl = cluster_factory(tile=tile)
    prob = KrigeProblem(cl, "c4", builtin_spec("matern-nugget", X, nu=0.5), y, theta)
    ll = prob.log_density()
    assert abs(ll - s["ll"]) <= 1e-10 * abs(s["ll"])
    Lh = prob._handles["L"]
    logdet = distla.log_det_from_chol(cl, Lh)
    assert abs(logdet - s["logdet"]) <= 1e-12 * abs(s["logdet"])
    L = cl.fetch(Lh.name)
    T = -(-n // tile)
    pad = T * tile - n  # this layout's identity-padded rows
    fro2 = float(torch.sum(L.data * L.data)) - pad
    assert np.sqrt(fro2 + (67320 - n)) == pytest.approx(s["norm_L_fro"], rel=1e-12)
    # leading block: the factor of a leading principal block is the leading block of L
    k = meta["c4_lead"]["k"]
    lead = _dense_lead(L, k)
    for x, want in zip(arr["c4_lead_x"], arr["c4_lead_Lx"]):
        got = (lead @ torch.from_numpy(x).to(lead.device)).cpu().numpy()
        assert relerr(got, want) <= 1e-9
    del lead
    # residual probe against a fresh copy of C
    C = distla.construct_distributed(cl, "c4.Cchk", "triangular", "gen.matern-nugget.cov", theta,
                                     inputs_name="c4.inputs", row_layout=prob.row_layout)
    Cd = cl.fetch(C.name)
    x = torch.zeros(T * tile, dtype=torch.float64, device=cl.device)
    x[:n] = torch.from_numpy(np.random.default_rng(8).standard_normal(n))
    t1, t2, cx = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    cl.call("bgp_tri_mv", p(L.data), n, tile, p(x), p(t1), 1, cl.stream)   # L^T x
    cl.call("bgp_tri_mv", p(L.data), n, tile, p(t1), p(t2), 0, cl.stream)  # L L^T x
    cl.call("bgp_tri_mv", p(Cd.data), n, tile, p(x), p(cx), 2, cl.stream)  # C x (lower stored)
    r = float(torch.linalg.norm((t2 - cx)[:n]) / torch.linalg.norm(cx[:n]))
    assert r <= 1e-13, r
