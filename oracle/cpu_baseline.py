"""Reference CPU timing of the likelihood path by operation-count sampling.

TEST / BASELINE INFRASTRUCTURE ONLY (imported by bench.py's `cpu_baseline`
and `--impl reference` legs).  It times the reference algorithm -- the P = 1
block sweep of bg/distla/kernels.py:35-75 (construct), 139-194 (Cholesky:
LAPACK potrf, trsm, BLAS-3 SYRK/GEMM on bs x bs blocks) and 200-250 (forward
solve) with the reference's default block size (bg/grid.py:108-113) -- on a
bounded sample of the real blocks of the n = 67,275 problem, and scales each
operation's mean time by its exact count in one evaluation:

  construct  B(B+1)/2 blocks           (single-threaded numpy, as reference)
  potrf      B                         (LAPACK, all host threads)
  trsm       B(B-1)/2                  (LAPACK)
  syrk       B(B-1)/2                  (BLAS-3, tril(W W^T))
  gemm       sum_J (B-J-1)(B-J-2)/2    (BLAS-3, A_RJ A_CJ^T)
  gemv       B(B-1)/2 + B trsv         (forward solve)

A full evaluation of the reference at n = 67,275 takes 4.6 min on the GPU
box's 16 host cores (oracle/full_eval.py, profiles/r02_cpu_full_eval.json);
the sample keeps bench.py within minutes and states itself in the JSON line.
SubEvalSampler (bench.py's sampler) measures the per-call times inside one
real evaluation of a prefix of the problem with the full problem's block
shapes; ReferenceSampler (isolated micro-timings) is kept for comparison.
"""

import math
import os
import time

import numpy as np
import scipy.linalg as la

from .blockgp_oracle import Generator, block_size, default_h


def op_counts(n, bs):
    B = math.ceil(n / bs)
    gemm = sum((B - J - 1) * (B - J - 2) // 2 for J in range(B))
    return {"construct": B * (B + 1) // 2, "potrf": B, "trsm": B * (B - 1) // 2,
            "syrk": B * (B - 1) // 2, "gemm": gemm, "gemv": B * (B - 1) // 2, "trsv": B}


def _construct_block(gen, theta, inputs, n, bs, I, J):
    """One block exactly as bg/distla/kernels.py:57-71 builds it."""
    r0, c0 = (I - 1) * bs + 1, (J - 1) * bs + 1
    jj, ii = np.meshgrid(np.arange(c0, c0 + bs), np.arange(r0, r0 + bs), indexing="xy")
    block = np.zeros((bs, bs))
    mask = (ii <= n) & (jj <= n)
    if I == J:
        mask &= ii >= jj
    block[mask] = np.asarray(gen(theta, inputs, ii[mask], jj[mask]), dtype=float)
    return block


class ReferenceSampler:
    """Times sampled reference operations on blocks of one problem."""

    def __init__(self, X, theta, nu=0.5, kernel="matern-nugget", seed=0):
        self.X = np.asarray(X, dtype=float)
        self.n = len(self.X)
        self.bs = block_size(self.n, default_h(self.n))
        self.B = math.ceil(self.n / self.bs)
        self.theta = np.asarray(theta, dtype=float)
        self.inputs = {"coords": self.X, "nu": nu}
        self.gen = Generator(f"gen.{kernel}.cov")
        self.rng = np.random.default_rng(seed)
        self.counts = op_counts(self.n, self.bs)
        # real blocks for the BLAS/LAPACK operations: a diagonal block and two
        # off-diagonal blocks of the covariance, and the factor of the former
        bs, B = self.bs, self.B
        self.A_diag = _construct_block(self.gen, self.theta, self.inputs, self.n, bs, 2, 2)
        self.A_diag = np.tril(self.A_diag) + np.tril(self.A_diag, -1).T
        self.L = la.cholesky(self.A_diag, lower=True)
        self.P1 = _construct_block(self.gen, self.theta, self.inputs, self.n, bs, B // 2, 2)
        self.P2 = _construct_block(self.gen, self.theta, self.inputs, self.n, bs, B - 1, 2)
        self.x = self.rng.standard_normal(bs)

    def sample(self, reps=6, construct_blocks=4):
        """One bounded sample; returns per-op mean seconds and wall time."""
        t0 = time.perf_counter()
        t = {}

        def clock(fn):
            fn()  # warm (thread pool spin-up); the reference runs these back to back
            fn()
            ts = []
            for _ in range(reps):
                s = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - s)
            return float(np.median(ts))

        A = self.A_diag
        t["potrf"] = clock(lambda: la.cholesky(A, lower=True, check_finite=False))
        t["trsm"] = clock(lambda: la.solve_triangular(self.L, self.P1.T, lower=True,
                                                      check_finite=False).T)
        C = self.P2.copy()
        t["gemm"] = clock(lambda: np.subtract(C, self.P1 @ self.P2.T, out=C))
        t["syrk"] = clock(lambda: np.subtract(C, np.tril(self.P1 @ self.P1.T), out=C))
        t["gemv"] = clock(lambda: self.P1 @ self.x)
        t["trsv"] = clock(lambda: la.solve_triangular(self.L, self.x, lower=True,
                                                      check_finite=False))
        tc = []
        for _ in range(construct_blocks):
            J = int(self.rng.integers(1, self.B + 1))
            I = int(self.rng.integers(J, self.B + 1))
            s = time.perf_counter()
            _construct_block(self.gen, self.theta, self.inputs, self.n, self.bs, I, J)
            tc.append(time.perf_counter() - s)
        t["construct"] = float(np.mean(tc))
        return t, time.perf_counter() - t0

    def extrapolate(self, t):
        """Seconds for one full evaluation and for the Cholesky alone."""
        c = self.counts
        chol = (c["potrf"] * t["potrf"] + c["trsm"] * t["trsm"] + c["syrk"] * t["syrk"]
                + c["gemm"] * t["gemm"])
        total = c["construct"] * t["construct"] + chol + c["gemv"] * t["gemv"] + c["trsv"] * t["trsv"]
        return total, chol

    def describe(self):
        return (f"reference P=1 block sweep (block {self.bs}, B={self.B}) at n={self.n}: "
                f"sampled real blocks per step (4 construct, median of 6 potrf/trsm/gemm/syrk/gemv/trsv), "
                f"scaled by exact op counts {self.counts}")


class SubEvalSampler:
    """The reference algorithm's per-operation times measured inside a real
    (smaller) evaluation: one full P = 1 evaluation (oracle/full_eval.py) on
    the first n_sub points with the FULL problem's block size, so every BLAS
    / LAPACK / construct call has the same shape as in the full run and runs
    back to back in the same sweep (streaming blocks, warm thread pools).
    Each kind's median call time is scaled by its exact count in the full
    evaluation (op_counts).  Isolated micro-timings (ReferenceSampler) were
    off by +24 % (median) / -37 % (min) against a timed full evaluation in
    this container; see DESIGN.md 6 for this sampler against the GPU box's
    timed full evaluations."""

    def __init__(self, X, theta, y=None, nu=0.5, kernel="matern-nugget", blocks=16, seed=0):
        self.X = np.asarray(X, dtype=float)
        self.n = len(self.X)
        self.bs = block_size(self.n, default_h(self.n))
        self.B = math.ceil(self.n / self.bs)
        self.n_sub = min(self.n, blocks * self.bs)
        self.theta = np.asarray(theta, dtype=float)
        self.kernel, self.nu = kernel, nu
        rng = np.random.default_rng(seed)
        self.y = np.asarray(y, dtype=float)[:self.n_sub] if y is not None else rng.standard_normal(self.n_sub)
        self.counts = op_counts(self.n, self.bs)

    def sample(self):
        from . import full_eval
        ot = {}
        t0 = time.perf_counter()
        full_eval.log_density(self.X[:self.n_sub], self.y, self.theta, kernel=self.kernel, nu=self.nu,
                              bs=self.bs, op_times=ot)
        # median call time per kind: a short run's first calls (thread pool
        # and page warm-up) would bias a mean upward
        t = {k: float(np.median(ot[k])) for k in ("construct", "potrf", "trsm", "syrk", "gemm", "gemv", "trsv")
             if ot.get(k)}
        return t, time.perf_counter() - t0

    extrapolate = ReferenceSampler.extrapolate

    def describe(self):
        return (f"reference P=1 block sweep (block {self.bs}, B={self.B}) at n={self.n}: per-call times "
                f"of each operation kind measured inside one full evaluation of the first {self.n_sub} "
                f"points (same block shapes), scaled by exact op counts {self.counts}")


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
