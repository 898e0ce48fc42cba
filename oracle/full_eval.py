"""One FULL evaluation of the reference algorithm at BASELINE config 4, timed.

TEST / BASELINE INFRASTRUCTURE ONLY (run by tools/cpu_full_eval.py on a GPU
box's host to validate the sampled CPU baseline of bench.py; never imported
by the product).  It is the reference's P = 1 path of
KrigeProblem.log_density (bg/gp/problem.py:119-142, 170-183) restated over
packed lower blocks so that n = 67,275 fits in ~19 GB (the oracle's dense
padded arrays would need 2 x 36 GB):

  construct   bg/distla/kernels.py:35-75 with the generator of
              bg/gp/kernels.py:42-46, 77-82 (numpy, single-threaded, as the
              reference), identity padding objects.py:60-80;
  Cholesky    bg/distla/kernels.py:139-194: per J, LAPACK potrf of A_JJ,
              TRSM A_IJ <- A_IJ L_JJ^-T, SYRK tril(W W^T) and GEMM-NT updates
              (BLAS on every host thread);
  solve       bg/distla/kernels.py:200-250 (GEMV partials in K order + TRSV);
  logdet / sumsq  kernels.py:493-522, block-ordered sums.

The block size is the reference's default (bg/grid.py:108-113: 990 at
n = 67,275).  Returns the log-likelihood and the phase times.
"""

import math
import time

import numpy as np
import scipy.linalg as la

from .blockgp_oracle import LOG_2PI, Generator, block_size, default_h


def _tri(I, J, B):
    """Packed index of lower block (I, J), 0-based, column-major."""
    return J * B - J * (J - 1) // 2 + (I - J)


def log_density(X, y, theta, kernel="matern-nugget", nu=0.5, bs=None, log=None, op_times=None):
    """One evaluation; with op_times (a dict) the wall time of every
    construct block / potrf / trsm / syrk / gemm / gemv / trsv call is
    appended per kind there (lists of seconds), for the sampled baseline."""
    tick = time.perf_counter
    acc = op_times if op_times is not None else {}

    def timed(kind, fn):
        t = tick()
        out = fn()
        acc.setdefault(kind, []).append(tick() - t)
        return out

    X = np.asarray(X, dtype=float)
    y = np.asarray(y, dtype=float)
    n = len(y)
    bs = bs or block_size(n, default_h(n))
    B = math.ceil(n / bs)
    gen = Generator(f"gen.{kernel}.cov")
    inputs = {"coords": X, "nu": nu}
    times = {}
    t0 = time.perf_counter()
    A = np.zeros((B * (B + 1) // 2, bs, bs))
    for J in range(B):
        for I in range(J, B):
            r0, c0 = I * bs + 1, J * bs + 1
            jj, ii = np.meshgrid(np.arange(c0, c0 + bs), np.arange(r0, r0 + bs), indexing="xy")
            mask = (ii <= n) & (jj <= n)
            if I == J:
                mask &= ii >= jj
            blk = A[_tri(I, J, B)]
            t = tick()
            blk[mask] = np.asarray(gen(theta, inputs, ii[mask], jj[mask]), dtype=float)
            acc.setdefault("construct", []).append(tick() - t)
    for t in range(n, B * bs):  # identity on the padded diagonal tail
        A[_tri(B - 1, B - 1, B)][t - (B - 1) * bs, t - (B - 1) * bs] = 1.0
    times["construct_s"] = time.perf_counter() - t0
    if log:
        log(f"construct {times['construct_s']:.1f} s")

    t1 = time.perf_counter()
    for J in range(B):
        L = timed("potrf", lambda: la.cholesky(A[_tri(J, J, B)], lower=True, check_finite=False))
        A[_tri(J, J, B)] = L
        for I in range(J + 1, B):
            k = _tri(I, J, B)
            A[k] = timed("trsm", lambda: la.solve_triangular(L, A[k].T, lower=True, check_finite=False).T)
        for C in range(J + 1, B):
            Wc = A[_tri(C, J, B)]
            for R in range(C, B):
                if R == C:
                    timed("syrk", lambda: np.subtract(A[_tri(R, C, B)], np.tril(Wc @ Wc.T),
                                                      out=A[_tri(R, C, B)]))
                else:
                    timed("gemm", lambda: np.subtract(A[_tri(R, C, B)], A[_tri(R, J, B)] @ Wc.T,
                                                      out=A[_tri(R, C, B)]))
        if log and J % 8 == 0:
            log(f"chol step {J}/{B} {time.perf_counter() - t1:.1f} s")
    times["cholesky_s"] = time.perf_counter() - t1

    t2 = time.perf_counter()
    resid = np.zeros(B * bs)
    resid[:n] = y
    u = np.zeros(B * bs)
    for J in range(B):
        r = resid[J * bs:(J + 1) * bs].copy()
        for K in range(J):
            r -= timed("gemv", lambda: A[_tri(J, K, B)] @ u[K * bs:(K + 1) * bs])
        u[J * bs:(J + 1) * bs] = timed("trsv", lambda: la.solve_triangular(
            A[_tri(J, J, B)], r, lower=True, check_finite=False))
    logdet = 0.0
    for J in range(B):
        live = min(max(n - J * bs, 0), bs)
        logdet += 2.0 * float(np.sum(np.log(np.diag(A[_tri(J, J, B)])[:live])))
    ssq = 0.0
    for J in range(B):
        lo, hi = J * bs, min((J + 1) * bs, n)
        ssq += float(np.dot(u[lo:hi], u[lo:hi]))
    times["solve_reduce_s"] = time.perf_counter() - t2
    times["eval_s"] = time.perf_counter() - t0
    ll = -0.5 * n * LOG_2PI - 0.5 * logdet - 0.5 * ssq
    return {"ll": ll, "logdet": logdet, "ssq": ssq, "block": bs, "B": B, **times}
