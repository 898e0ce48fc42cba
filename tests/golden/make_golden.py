"""Generate golden fixtures by running the REFERENCE blockgp package.

Run in the build container only (needs /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden_small.npz (arrays) and golden_scalars.json.
Every value comes from the reference's own public API (spawn / distla /
KrigeProblem) on seeded inputs; the oracle (oracle/blockgp_oracle.py) and the
CUDA path are both checked against these files by tests/.  The C4 inputs
(n = 67,275) are produced separately by make_c4_inputs.py.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from blockgp import distla, spawn  # noqa: E402
from blockgp.errors import NotPositiveDefinite, SingularDiagonal  # noqa: E402
from blockgp.gp import KrigeProblem, builtin_spec  # noqa: E402
from blockgp.gp import kernels as gpk  # noqa: E402
from blockgp.gp.problem import CovarianceSpec  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.blockgp_oracle import config_inputs, dense_cov  # noqa: E402

# config-5 kernel through the reference's own extension point
# (bg/gp/kernels.py:68-98)
gpk._make_pairwise("sqexp-nugget", gpk._sqexp_corr)


def spd_matrix(n, seed=0):
    """tests/conftest.py:24-28 of the reference."""
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((n, n))
    return B @ B.T + n * np.eye(n)


def main():
    arrays, scalars = {}, {}
    cl = spawn(1, seed=0)
    try:
        # --- construct: every built-in generator on 2-D coords ------------
        rng = np.random.default_rng(100)
        X = rng.uniform(0, 1, (37, 2))
        Xp = rng.uniform(0, 1, (11, 2))
        arrays["con_X"], arrays["con_Xp"] = X, Xp
        rows = distla.make_layout(37, cl.grid, h=2)     # block 19, padded 38
        cols = distla.make_layout(11, cl.grid, h=1)
        cases = {
            "matern05": ("matern-nugget", [1.3, 0.3, 0.05], {"nu": 0.5}),
            "matern15": ("matern-nugget", [2.0, 0.2, 0.05], {"nu": 1.5}),
            "matern25": ("matern-nugget", [0.7, 0.25, 0.1], {"nu": 2.5}),
            "maternnn": ("matern", [1.1, 0.4], {"nu": 1.5}),
            "sqexp": ("sqexp", [1.4, 0.3], {}),
            "sqexpnug": ("sqexp-nugget", [1.0, 0.02, 0.1], {}),
            "white": ("white", [2.5], {}),
            "product": ("matern-product-nugget", [1.2, 0.3, 0.2, 0.15],
                        {"nu1": 0.5, "nu2": 1.5}),
        }
        for key, (kern, theta, extra) in cases.items():
            inputs = {"coords": X, "pred_coords": Xp}
            inputs.update(extra)
            cl.push("inp", inputs)
            t = distla.construct_distributed(cl, "C", "triangular",
                                             f"gen.{kern}.cov", theta,
                                             inputs_name="inp", row_layout=rows)
            arrays[f"con_{key}_cov"] = distla.collect(cl, t)
            r = distla.construct_distributed(cl, "Cx", "rectangular",
                                             f"gen.{kern}.cross", theta,
                                             inputs_name="inp", row_layout=rows,
                                             col_layout=cols)
            arrays[f"con_{key}_cross"] = distla.collect(cl, r)
            p = distla.construct_distributed(cl, "Cp", "triangular",
                                             f"gen.{kern}.pred", theta,
                                             inputs_name="inp", row_layout=cols)
            arrays[f"con_{key}_pred"] = distla.collect(cl, p)
            v = distla.construct_distributed(cl, "pv", "vector",
                                             f"gen.{kern}.predvar", theta,
                                             inputs_name="inp", row_layout=cols)
            arrays[f"con_{key}_predvar"] = distla.collect(cl, v)
            scalars[f"con_{key}"] = {"kernel": kern, "theta": theta,
                                     "inputs": extra}

        # --- Cholesky / solves / products on spd_matrix ---------------------
        for n, h in ((37, 2), (257, 2), (300, 1)):
            A = spd_matrix(n, seed=n)
            b = np.random.default_rng(n + 1).standard_normal(n)
            R = np.random.default_rng(n + 2).standard_normal((n, 7))
            lay = distla.make_layout(n, cl.grid, h=h)
            lc = distla.make_layout(7, cl.grid, h=1)
            C = distla.distribute(cl, "C", A, "triangular", lay)
            L, _ = distla.distributed_cholesky(cl, C, "L")
            bd = distla.distribute(cl, "b", b, "vector", lay)
            u = distla.triangular_solve(cl, L, bd, "u", side="forward")
            x = distla.triangular_solve(cl, L, u, "x", side="back")
            Rd = distla.distribute(cl, "R", R, "rectangular", lay, lc)
            W = distla.triangular_solve(cl, L, Rd, "W", side="forward")
            Wb = distla.triangular_solve(cl, L, Rd, "Wb", side="back")
            w = distla.crossprod_mat_vec(cl, W, u, "w")
            S = distla.crossprod_self(cl, W, "S")
            d = distla.crossprod_self_diag(cl, W, "d")
            k = f"la{n}"
            arrays.update({f"{k}_A": A, f"{k}_b": b, f"{k}_R": R,
                           f"{k}_L": distla.collect(cl, L),
                           f"{k}_u": distla.collect(cl, u),
                           f"{k}_x": distla.collect(cl, x),
                           f"{k}_W": distla.collect(cl, W),
                           f"{k}_Wb": distla.collect(cl, Wb),
                           f"{k}_w": distla.collect(cl, w),
                           f"{k}_S": distla.collect(cl, S),
                           f"{k}_d": distla.collect(cl, d)})
            scalars[k] = {"h": h, "block": lay.block_size,
                          "logdet": distla.log_det_from_chol(cl, L),
                          "ssq": distla.sum_squares(cl, u)}

        # --- error semantics -------------------------------------------------
        lay = distla.make_layout(6, cl.grid, h=1)
        C = distla.distribute(cl, "C", -np.eye(6), "triangular", lay)
        try:
            distla.distributed_cholesky(cl, C, "L")
        except NotPositiveDefinite as exc:
            scalars["npd_minus_identity_block"] = exc.block_index
        A = spd_matrix(40, seed=3)
        A[25, 25] = -50.0                     # indefinite inside block 2 (h=2)
        lay = distla.make_layout(40, cl.grid, h=2)
        C = distla.distribute(cl, "C", A, "triangular", lay)
        arrays["npd_A"] = A
        try:
            distla.distributed_cholesky(cl, C, "L")
        except NotPositiveDefinite as exc:
            scalars["npd_A_block_h2"] = exc.block_index
        lay = distla.make_layout(2, cl.grid, h=1)
        L = distla.distribute(cl, "L", [[1.0, 0.0], [1.0, 0.0]], "triangular", lay)
        b = distla.distribute(cl, "b", [1.0, 1.0], "vector", lay)
        try:
            distla.triangular_solve(cl, L, b, "x", side="forward")
        except SingularDiagonal:
            scalars["singular_detected"] = True
    finally:
        cl.shutdown()

    # --- GP end to end (2-D, reference KrigeProblem) ------------------------
    for key, (n, m, kern, theta, extra, seed) in {
        "gp400": (400, 25, "matern-nugget", [1.5, 0.2, 0.1], {"nu": 0.5}, 3),
        "gp300m15": (300, 16, "matern-nugget", [2.0, 0.1, 0.05], {"nu": 1.5}, 4),
        "gp250m25": (250, 9, "matern-nugget", [0.9, 0.15, 0.02], {"nu": 2.5}, 5),
        "gp300sq": (300, 12, "sqexp-nugget", [1.0, 0.05, 0.1], {}, 6),
    }.items():
        rng = np.random.default_rng(seed)
        X = rng.uniform(0, 1, (n, 2))
        Xp = rng.uniform(0, 1, (m, 2))
        theta = np.array(theta)
        C = dense_cov(kern, theta, X, **extra)
        y = np.linalg.cholesky(C) @ rng.standard_normal(n)
        if kern == "sqexp-nugget":
            inputs = {"coords": X, "pred_coords": Xp}
            spec = CovarianceSpec(cov_fn="gen.sqexp-nugget.cov",
                                  cross_cov_fn="gen.sqexp-nugget.cross",
                                  pred_cov_fn="gen.sqexp-nugget.pred",
                                  pred_var_fn="gen.sqexp-nugget.predvar",
                                  inputs=inputs, n_params=3)
        else:
            spec = builtin_spec(kern, X, Xp, **extra)
        for P, h in ((1, 1), (3, 2)):
            cl = spawn(P, seed=0)
            try:
                prob = KrigeProblem(cl, "g", spec, y, theta, m=m, h_n=h, h_m=1)
                ll = prob.log_density()
                mean, se = prob.predict(se_fit=True)
                PV = prob.prediction_variance()
            finally:
                cl.shutdown()
            if P == 1:
                arrays.update({f"{key}_X": X, f"{key}_Xp": Xp, f"{key}_y": y,
                               f"{key}_mean": mean, f"{key}_se": se,
                               f"{key}_PV": PV})
                scalars[key] = {"kernel": kern, "theta": list(theta),
                                "inputs": extra, "ll": ll}
            else:
                scalars[key]["ll_P3h2"] = ll

    # --- C1 (BASELINE config 1) full: reference ll on the 8d recipe ---------
    kern, X, theta, extra, z = config_inputs(1)
    C = dense_cov(kern, theta, X, **extra)
    y = np.linalg.cholesky(C) @ z
    cl = spawn(1, seed=0)
    try:
        spec = builtin_spec(kern, X, **extra)
        prob = KrigeProblem(cl, "c1", spec, y, theta)
        ll = prob.log_density()
        L = prob._handles["L"]
        logdet = distla.log_det_from_chol(cl, L)
        ssq = distla.sum_squares(cl, prob._handles["u"])
        ucol = distla.collect(cl, prob._handles["u"])
    finally:
        cl.shutdown()
    arrays["c1_y"] = y
    arrays["c1_u"] = ucol
    scalars["c1"] = {"ll": ll, "logdet": logdet, "ssq": ssq,
                     "survey_ll": -1235.1310506672912}

    # --- C2 (10 range values) at reduced n = 2048 (same recipe) -------------
    kern, X, theta, extra, z = config_inputs(2, n=2048)
    C = dense_cov(kern, theta, X, **extra)
    y = np.linalg.cholesky(C) @ z
    cl = spawn(1, seed=0)
    try:
        spec = builtin_spec(kern, X, **extra)
        prob = KrigeProblem(cl, "c2", spec, y, theta)
        lls = [prob.log_density(np.array([2.0, r, 0.05]))
               for r in np.linspace(0.02, 0.2, 10)]
    finally:
        cl.shutdown()
    arrays["c2s_y"] = y
    scalars["c2_n2048"] = {"ll": lls}

    # --- simulation (rank streams, bg/rng.py; P = 1) ---------------------
    from blockgp.rng import RankStream
    arrays["rng_seed21_rank1"] = RankStream(21, 1).standard_normals(1000)
    rng = np.random.default_rng(21)
    X = rng.uniform(0, 1, (60, 2))
    Xp = rng.uniform(0, 1, (9, 2))
    theta = np.array([1.3, 0.3, 0.1])
    y = np.linalg.cholesky(dense_cov("matern-nugget", theta, X, nu=0.5)) @ rng.standard_normal(60)
    cl = spawn(1, seed=21)
    try:
        spec = builtin_spec("matern-nugget", X, Xp, nu=0.5)
        prob = KrigeProblem(cl, "s", spec, y, theta, m=9)
        arrays["sim_unc"] = prob.simulate_realizations(4, post=False)
        arrays["sim_post"] = prob.simulate_realizations(3, post=True)
        arrays["sim_unc2"] = prob.simulate_realizations(2, post=False)
    finally:
        cl.shutdown()
    arrays.update({"sim_X": X, "sim_Xp": Xp, "sim_y": y})
    scalars["sim"] = {"seed": 21, "theta": list(theta), "nu": 0.5}

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **arrays)
    with open(os.path.join(HERE, "golden_scalars.json"), "w") as f:
        json.dump(scalars, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(scalars), "scalar groups")
    print("C1 ll", scalars["c1"]["ll"], "survey", scalars["c1"]["survey_ll"])


if __name__ == "__main__":
    main()
