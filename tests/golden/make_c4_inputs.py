"""Freeze the BASELINE config-4 inputs (n = 67,275): coords X and y = L z.

Recipe: SURVEY.md section 8d (seed 0, 10 % jittered duplicates, exponential
covariance theta = (1.0, 0.08, 0.02)).  L is LAPACK dpotrf (OpenBLAS) of the
dense covariance built with the reference generator formula
(bg/gp/kernels.py:16-29, 42-46, 77-82).  Needs ~37 GB RAM and ~10 min on 8
cores; run once in the build container:

    python tests/golden/make_c4_inputs.py

Writes tests/golden/c4_inputs.npz (X, y, z) and c4_scalars.json (logdet,
||y||, ||z||^2, ||L||_F of this factor) for comparison with BASELINE.md 3.
"""

import json
import os
import sys
import time

import numpy as np
import scipy.linalg as la

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.blockgp_oracle import config_inputs  # noqa: E402


def main():
    kern, X, theta, extra, z = config_inputs(4)
    n = len(X)
    t0 = time.time()
    A = np.empty((n, n))            # C order; only the lower triangle is filled
    chunk = 512
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        dx = X[r0:r1, None, 0] - X[None, :r1, 0]
        dy = X[r0:r1, None, 1] - X[None, :r1, 1]
        d = np.sqrt(dx * dx + dy * dy)
        blk = theta[0] * np.exp(-(np.sqrt(2.0 * 0.5) * d / theta[1]))
        idx = np.arange(r0, r1)
        blk[idx - r0, idx] += theta[2]
        A[r0:r1, :r1] = blk
    print("built", time.time() - t0, flush=True)
    # In-place right-looking block Cholesky of the lower triangle (LAPACK on
    # the diagonal blocks, BLAS-3 trailing updates).  A single dpotrf call is
    # not usable: LP64 LAPACK index arithmetic overflows past 2^31 elements.
    bs = 4096
    for j0 in range(0, n, bs):
        j1 = min(n, j0 + bs)
        Ljj = la.cholesky(A[j0:j1, j0:j1], lower=True, check_finite=False)
        A[j0:j1, j0:j1] = Ljj
        if j1 < n:
            P = la.solve_triangular(Ljj, A[j1:, j0:j1].T, lower=True,
                                    check_finite=False).T
            A[j1:, j0:j1] = P
            for c0 in range(j1, n, bs):
                c1 = min(n, c0 + bs)
                A[c0:, c0:c1] -= P[c0 - j1:] @ P[c0 - j1:c1 - j1].T
        print("col", j0, time.time() - t0, flush=True)
    print("factored", time.time() - t0, flush=True)
    y = np.zeros(n)
    for r0 in range(0, n, bs):
        r1 = min(n, r0 + bs)
        y[r0:r1] = np.tril(A[r0:r1, :r1], r0) @ z[:r1]
    diag = np.diagonal(A).copy()
    logdet = 2.0 * float(np.sum(np.log(diag)))
    fro2 = 0.0
    for r0 in range(0, n, 4096):
        r1 = min(n, r0 + 4096)
        blk = A[r0:r1, :r1]
        fro2 += float(np.sum(np.tril(blk, r0) ** 2))
    out = {"n": n, "logdet": logdet, "norm_y": float(np.linalg.norm(y)),
           "ssq_z": float(z @ z), "norm_L_fro": fro2 ** 0.5,
           "survey": {"ll": -5184.4952498986895, "logdet": -180826.2576652042,
                      "ssq": 67552.06852231288, "norm_L_fro": 262.04102732205894,
                      "norm_y": 282.16573588901014}}
    out["ll_from_this_factor"] = (-0.5 * n * np.log(2 * np.pi) - 0.5 * logdet
                                  - 0.5 * out["ssq_z"])
    np.savez_compressed(os.path.join(HERE, "c4_inputs.npz"), X=X, y=y, z=z)
    with open(os.path.join(HERE, "c4_scalars.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1), time.time() - t0)


if __name__ == "__main__":
    main()
