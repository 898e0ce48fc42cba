"""Freeze REFERENCE outputs at the full BASELINE config sizes.

Run in the build container only (needs /root/reference, read-only; ~10 min
and ~25 GB RAM on 8 cores):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_full_configs.py

Every value comes from the reference's own public API (spawn / distla /
KrigeProblem, P = 1, default h) on the SURVEY.md 8d recipe:

  * C2: n = 16,384 Matern 3/2, the ten log-likelihoods at
    rho = linspace(0.02, 0.2, 10) (bg/gp/problem.py:170-183);
  * C3: n = 32,768, m = 4,096: log_density and the full kriging mean and se
    vectors of predict(se_fit=True) (bg/gp/problem.py:221-244);
  * C5's kernel (squared exponential + nugget, registered through the
    reference's own _make_pairwise, bg/gp/kernels.py:68-98) at n = 16,384:
    ll, logdet, ssq;
  * C4's leading 4,096 x 4,096 block of L (the Cholesky factor of a leading
    principal block is the leading block of the full factor): two seeded
    probes L x, so the -m gpu suite can check the full-size factor
    normwise without an 18 GB fixture.

Coordinates are regenerated from the seed by oracle.config_inputs (numpy's
PCG64 stream is stable); their checksums are frozen next to the outputs so
a drifting generator fails loudly.  y = L(theta) z uses LAPACK on the dense
covariance (any correct FP64 factor: SURVEY.md 8c slack test).

Writes tests/golden/full_configs.npz and full_configs.json.
"""

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from blockgp import distla, spawn  # noqa: E402
from blockgp.gp import KrigeProblem, builtin_spec  # noqa: E402
from blockgp.gp import kernels as gpk  # noqa: E402
from blockgp.gp.problem import CovarianceSpec  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.blockgp_oracle import c3_pred_coords, config_inputs, dense_cov  # noqa: E402

gpk._make_pairwise("sqexp-nugget", gpk._sqexp_corr)

C2_RHO = np.linspace(0.02, 0.2, 10)


def checksum(X):
    return {"sum": float(np.sum(X)), "sumsq": float(np.sum(X * X)),
            "first": [float(v) for v in X.ravel()[:4]]}


def blocked_cholesky(A, bs=4096):
    """In-place right-looking block Cholesky of the lower triangle (LAPACK on
    the diagonal blocks, BLAS-3 updates): one dpotrf call on a 32,768-point
    covariance crashes inside OpenBLAS here."""
    import scipy.linalg as la
    n = len(A)
    for j0 in range(0, n, bs):
        j1 = min(n, j0 + bs)
        Ljj = la.cholesky(A[j0:j1, j0:j1], lower=True, check_finite=False)
        A[j0:j1, j0:j1] = Ljj
        if j1 < n:
            P = la.solve_triangular(Ljj, A[j1:, j0:j1].T, lower=True, check_finite=False).T
            A[j1:, j0:j1] = P
            for c0 in range(j1, n, bs):
                c1 = min(n, c0 + bs)
                A[c0:, c0:c1] -= P[c0 - j1:] @ P[c0 - j1:c1 - j1].T
    return np.tril(A)


def simulate(kern, X, theta, extra, z):
    C = dense_cov(kern, theta, X, **extra)
    L = np.linalg.cholesky(C) if len(X) <= 16384 else blocked_cholesky(C)
    y = L @ z
    del C, L
    return y


CACHE = "/tmp/golden_full"


def cached(key, fn):
    """Per-config results cached under /tmp so an interrupted run resumes."""
    import pickle
    os.makedirs(CACHE, exist_ok=True)
    path = os.path.join(CACHE, key + ".pkl")
    if os.path.exists(path):
        with open(path, "rb") as f:
            return pickle.load(f)
    out = fn()
    with open(path, "wb") as f:
        pickle.dump(out, f)
    return out


def main():
    arrays, meta = {}, {}
    t0 = time.time()

    # --- C2 -------------------------------------------------------------
    def c2():
        kern, X, theta, extra, z = config_inputs(2)
        y = simulate(kern, X, theta, extra, z)
        cl = spawn(1, seed=0)
        try:
            prob = KrigeProblem(cl, "c2", builtin_spec(kern, X, **extra), y, theta)
            lls = [prob.log_density(np.array([2.0, r, 0.05])) for r in C2_RHO]
        finally:
            cl.shutdown()
        return {"c2_y": y}, {"n": len(X), "X": checksum(X), "rho": [float(r) for r in C2_RHO],
                             "ll": lls}
    a, meta["c2"] = cached("c2", c2)
    arrays.update(a)
    print("C2", meta["c2"]["ll"], time.time() - t0, flush=True)

    # --- C3 -------------------------------------------------------------
    def c3():
        kern, X, theta, extra, z = config_inputs(3)
        Xp = c3_pred_coords()
        y = simulate(kern, X, theta, extra, z)
        cl = spawn(1, seed=0)
        try:
            prob = KrigeProblem(cl, "c3", builtin_spec(kern, X, Xp, **extra), y, theta, m=len(Xp))
            ll = prob.log_density()
            mean, se = prob.predict(se_fit=True)
        finally:
            cl.shutdown()
        return ({"c3_y": y, "c3_mean": mean, "c3_se": se},
                {"n": len(X), "m": len(Xp), "X": checksum(X), "ll": ll,
                 "norm_mean": float(np.linalg.norm(mean)), "norm_se": float(np.linalg.norm(se))})
    a, meta["c3"] = cached("c3", c3)
    arrays.update(a)
    print("C3", meta["c3"], time.time() - t0, flush=True)

    # --- C5's kernel at n = 16,384 ----------------------------------------
    def c5s():
        kern, X, theta, extra, z = config_inputs(5, n=16384)
        y = simulate(kern, X, theta, extra, z)
        spec = CovarianceSpec(cov_fn="gen.sqexp-nugget.cov", cross_cov_fn="gen.sqexp-nugget.cross",
                              pred_cov_fn="gen.sqexp-nugget.pred",
                              pred_var_fn="gen.sqexp-nugget.predvar",
                              inputs={"coords": X}, n_params=3)
        cl = spawn(1, seed=0)
        try:
            prob = KrigeProblem(cl, "c5s", spec, y, theta)
            ll = prob.log_density()
            logdet = distla.log_det_from_chol(cl, prob._handles["L"])
            ssq = distla.sum_squares(cl, prob._handles["u"])
        finally:
            cl.shutdown()
        return {"c5s_y": y}, {"n": len(X), "X": checksum(X), "theta": [float(t) for t in theta],
                              "ll": ll, "logdet": logdet, "ssq": ssq}
    a, meta["c5s"] = cached("c5s", c5s)
    arrays.update(a)
    print("C5 kernel n=16384", meta["c5s"], time.time() - t0, flush=True)

    # --- C4's leading block of L -------------------------------------------
    def c4lead():
        kern, X, theta, extra, _ = config_inputs(4)
        k = 4096
        cl = spawn(1, seed=0)
        try:
            cl.push("inp", {"coords": X[:k], **extra})
            rows = distla.make_layout(k, cl.grid)
            C = distla.construct_distributed(cl, "C", "triangular", f"gen.{kern}.cov", theta,
                                             inputs_name="inp", row_layout=rows)
            L, _ = distla.distributed_cholesky(cl, C, "L")
            Lk = distla.collect(cl, L)
        finally:
            cl.shutdown()
        probes = np.random.default_rng(44).standard_normal((2, k))
        return ({"c4_lead_x": probes, "c4_lead_Lx": np.stack([Lk @ x for x in probes])},
                {"k": k, "X": checksum(X), "norm_L_fro_lead": float(np.linalg.norm(Lk))})
    a, meta["c4_lead"] = cached("c4lead", c4lead)
    arrays.update(a)
    print("C4 lead", meta["c4_lead"], time.time() - t0, flush=True)

    np.savez(os.path.join(HERE, "full_configs.npz"), **arrays)
    with open(os.path.join(HERE, "full_configs.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
