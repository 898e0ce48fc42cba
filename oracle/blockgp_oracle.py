"""CPU oracle for the bigGP / blockgp Gaussian-process likelihood path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module,
and only as the checker or the timed CPU baseline.  The product path
(`paper_1305_4886_b200`) never imports it and has no CPU fallback.

This is a numpy/scipy restatement of the reference's algorithm at P = 1 (one
worker owns every block), following `/root/reference/pkg/src/blockgp/`
(abbreviated `bg/` below) function by function:

  generators      bg/gp/kernels.py:16-34 (Matern 1/2, 3/2, 5/2; sqexp),
                  42-46 (_dist), 68-98 (_make_pairwise: cov/cross/pred/predvar),
                  114-172 (product, white)
  construct       bg/distla/kernels.py:35-75 + bg/distla/objects.py:60-80
  cholesky        bg/distla/kernels.py:139-194 (right-looking block sweep)
  solve_vector    bg/distla/kernels.py:200-250
  solve_rect      bg/distla/kernels.py:253-307
  xprod_*         bg/distla/kernels.py:387-487
  logdet, sumsq   bg/distla/kernels.py:493-522, bg/distla/__init__.py:154-162
  log_density     bg/gp/problem.py:119-142, 170-183
  predict         bg/gp/problem.py:144-167, 221-244
  pred. variance  bg/gp/problem.py:246-265

The arithmetic goes through the same third-party routines the reference uses
(numpy `@`, scipy.linalg.cholesky / solve_triangular -> OpenBLAS/LAPACK), on
the same block schedule, so at equal block size the results agree with the
reference to the last few ulps.  Parity pin: `tests/test_oracle.py` checks this
module against fixtures produced by the reference itself
(`tests/golden/make_golden.py`) and against the survey's scalar goldens.
"""

import math

import numpy as np
import scipy.linalg as la

LOG_2PI = float(np.log(2.0 * np.pi))
HALF_INTEGER_NU = (0.5, 1.5, 2.5)


class OracleNotPD(Exception):
    """Non-positive pivot; `block_index` is 1-based (bg/distla/kernels.py:146-148)."""

    def __init__(self, block_index):
        self.block_index = block_index
        super().__init__(f"not positive definite at diagonal block {block_index}")


class OracleSingular(Exception):
    """Zero / non-positive diagonal (bg/distla/kernels.py:245-246, 506-507)."""


# ---------------------------------------------------------------------------
# correlation functions and generators


def matern_correlation(d, rho, nu):
    """bg/gp/kernels.py:16-29."""
    d = np.asarray(d, dtype=float)
    if rho <= 0:
        raise ValueError(f"range must be positive, got {rho}")
    s = np.sqrt(2.0 * nu) * d / rho
    if nu == 0.5:
        return np.exp(-s)
    if nu == 1.5:
        return (1.0 + s) * np.exp(-s)
    if nu == 2.5:
        return (1.0 + s + s * s / 3.0) * np.exp(-s)
    raise ValueError(f"nu={nu} not supported")


def sqexp_correlation(d, rho):
    """bg/gp/kernels.py:32-34."""
    d = np.asarray(d, dtype=float)
    return np.exp(-0.5 * (d / rho) ** 2)


def _points(X):
    X = np.asarray(X, dtype=float)
    return X[:, None] if X.ndim == 1 else X


def _dist(X, Y, i, j):
    """bg/gp/kernels.py:42-46 (1-based i, j)."""
    diff = X[i - 1] - Y[j - 1]
    return np.sqrt(np.sum(diff * diff, axis=-1))


class Generator:
    """One entrywise generator id of bg/gp/kernels.py, evaluated on the CPU.

    `family` in {"matern", "matern-nugget", "sqexp", "sqexp-nugget",
    "white", "matern-product-nugget", "delta", "linear_index", "zero"}, `part`
    in {"cov", "cross", "pred", "predvar"}.  "sqexp-nugget" is the config-5
    kernel registered through the reference's `_make_pairwise` extension point
    (bg/gp/kernels.py:68-98).
    """

    def __init__(self, gen_id):
        self.gen_id = gen_id
        parts = gen_id.split(".")
        if len(parts) == 2:
            self.family, self.part = parts[1], None
        else:
            self.family, self.part = parts[1], parts[2]

    def __call__(self, params, inputs, i, j=None):
        fam, part = self.family, self.part
        params = np.asarray(params, dtype=float)
        if fam == "zero":
            return np.zeros(len(i))
        if fam == "delta":
            return (i == j).astype(float)
        if fam == "linear_index":
            return i + inputs["n"] * (j - 1.0)
        if part == "predvar":
            return np.full(len(i), params[0])
        if fam == "white":
            if part == "cross":
                return np.zeros(len(i))
            return params[0] * (i == j)
        left, right = {"cov": ("coords", "coords"),
                       "cross": ("coords", "pred_coords"),
                       "pred": ("pred_coords", "pred_coords")}[part]
        X, Y = _points(inputs[left]), _points(inputs[right])
        if fam == "matern-product-nugget":
            # bg/gp/kernels.py:114-148
            d1 = np.abs(X[i - 1, 0] - Y[j - 1, 0])
            d2 = np.abs(X[i - 1, 1] - Y[j - 1, 1])
            k = params[0] * (matern_correlation(d1, params[1], inputs.get("nu1", 0.5))
                             * matern_correlation(d2, params[2], inputs.get("nu2", 0.5)))
            if part == "cov":
                k = k + params[3] * (i == j)
            return k
        d = _dist(X, Y, i, j)
        if fam.startswith("sqexp"):
            corr = sqexp_correlation(d, params[1])
        else:
            corr = matern_correlation(d, params[1], inputs.get("nu", 0.5))
        k = params[0] * corr
        if part == "cov" and fam.endswith("-nugget"):
            k = k + params[-1] * (i == j)
        return k


# ---------------------------------------------------------------------------
# block layout (bg/grid.py:77-113) at P = 1


def block_size(n, h, D=1):
    return math.ceil(n / (h * D))


def default_h(n, D=1, target=1000):
    """bg/grid.py:108-113."""
    h = 1
    while math.ceil(n / (h * D)) > target:
        h += 1
    return h


# ---------------------------------------------------------------------------
# construction: dense padded arrays built block by block


def construct_triangular(gen, params, inputs, n, bs):
    """bg/distla/kernels.py:35-75 + objects.py:60-80 for a triangular object.

    Returns the padded dense lower-triangular array (padded_n x padded_n) with
    the identity on the padded diagonal tail and zeros above the diagonal.
    """
    B = math.ceil(n / bs)
    pn = B * bs
    A = np.zeros((pn, pn))
    for J in range(1, B + 1):
        for I in range(J, B + 1):
            r0, c0 = (I - 1) * bs + 1, (J - 1) * bs + 1
            jj, ii = np.meshgrid(np.arange(c0, c0 + bs), np.arange(r0, r0 + bs),
                                 indexing="xy")
            mask = (ii <= n) & (jj <= n)
            if I == J:
                mask &= ii >= jj
            block = np.zeros((bs, bs))
            block[mask] = np.asarray(gen(params, inputs, ii[mask], jj[mask]),
                                     dtype=float)
            A[r0 - 1:r0 - 1 + bs, c0 - 1:c0 - 1 + bs] = block
    for t in range(n, pn):
        A[t, t] = 1.0
    return A


def construct_rectangular(gen, params, inputs, n, m, bs_r, bs_c):
    """bg/distla/kernels.py:35-75 for a rectangular object (zero padding)."""
    Br, Bc = math.ceil(n / bs_r), math.ceil(m / bs_c)
    A = np.zeros((Br * bs_r, Bc * bs_c))
    for J in range(1, Bc + 1):
        for I in range(1, Br + 1):
            r0, c0 = (I - 1) * bs_r + 1, (J - 1) * bs_c + 1
            jj, ii = np.meshgrid(np.arange(c0, c0 + bs_c), np.arange(r0, r0 + bs_r),
                                 indexing="xy")
            mask = (ii <= n) & (jj <= m)
            block = np.zeros((bs_r, bs_c))
            block[mask] = np.asarray(gen(params, inputs, ii[mask], jj[mask]),
                                     dtype=float)
            A[r0 - 1:r0 - 1 + bs_r, c0 - 1:c0 - 1 + bs_c] = block
    return A


def construct_vector(gen, params, inputs, n, bs):
    """bg/distla/kernels.py:46-55 (3-argument generator, zero padding)."""
    pn = math.ceil(n / bs) * bs
    x = np.zeros(pn)
    i = np.arange(1, n + 1)
    x[:n] = np.asarray(gen(params, inputs, i), dtype=float)
    return x


def pad_triangular(A, n, bs):
    """bg/distla/objects.py:83-105 (split_array, triangular)."""
    pn = math.ceil(n / bs) * bs
    P = np.zeros((pn, pn))
    P[:n, :n] = np.tril(np.asarray(A, dtype=float))
    for t in range(n, pn):
        P[t, t] = 1.0
    return P


# ---------------------------------------------------------------------------
# Cholesky and solves on padded dense arrays, block schedule of P = 1


def cholesky(A, bs):
    """Right-looking block Cholesky, bg/distla/kernels.py:139-194 at P = 1.

    `A` is the padded lower-triangular array; factored in a copy.  Raises
    OracleNotPD(J) at the first diagonal block whose LAPACK potrf fails.
    """
    A = np.array(A, dtype=float, copy=True)
    pn = A.shape[0]
    B = pn // bs
    blk = lambda I, J: (slice((I - 1) * bs, I * bs), slice((J - 1) * bs, J * bs))
    for J in range(1, B + 1):
        try:
            L = la.cholesky(A[blk(J, J)], lower=True, check_finite=False)
        except la.LinAlgError:
            raise OracleNotPD(J) from None
        A[blk(J, J)] = L
        for I in range(J + 1, B + 1):
            A[blk(I, J)] = la.solve_triangular(L, A[blk(I, J)].T, lower=True,
                                               check_finite=False).T
        for C in range(J + 1, B + 1):
            for R in range(C, B + 1):
                if R == C:
                    W = A[blk(R, J)]
                    A[blk(R, C)] -= np.tril(W @ W.T)
                else:
                    A[blk(R, C)] -= A[blk(R, J)] @ A[blk(C, J)].T
    return A


def solve_vector(L, b, bs, forward=True):
    """bg/distla/kernels.py:200-250: blocked substitution, partials in K order."""
    pn = L.shape[0]
    B = pn // bs
    b = np.asarray(b, dtype=float)
    x = np.zeros(pn)
    order = range(1, B + 1) if forward else range(B, 0, -1)
    sl = lambda J: slice((J - 1) * bs, J * bs)
    for J in order:
        Ks = range(1, J) if forward else range(J + 1, B + 1)
        acc = b[sl(J)].copy()
        for K in Ks:
            Lb = L[sl(J), sl(K)] if forward else L[sl(K), sl(J)]
            acc -= (Lb @ x[sl(K)]) if forward else (Lb.T @ x[sl(K)])
        Ljj = L[sl(J), sl(J)]
        if np.any(np.diag(Ljj) == 0.0):
            raise OracleSingular(f"zero diagonal in block {J}")
        x[sl(J)] = la.solve_triangular(Ljj, acc, lower=True,
                                       trans=0 if forward else 1,
                                       check_finite=False)
    return x


def solve_rect(L, Bm, bs, forward=True):
    """bg/distla/kernels.py:253-307 with all RHS columns in one block column."""
    pn = L.shape[0]
    B = pn // bs
    Bm = np.asarray(Bm, dtype=float)
    X = np.zeros_like(Bm)
    order = range(1, B + 1) if forward else range(B, 0, -1)
    sl = lambda J: slice((J - 1) * bs, J * bs)
    for J in order:
        Ks = range(1, J) if forward else range(J + 1, B + 1)
        acc = Bm[sl(J)].copy()
        for K in Ks:
            Lb = L[sl(J), sl(K)] if forward else L[sl(K), sl(J)]
            acc -= (Lb @ X[sl(K)]) if forward else (Lb.T @ X[sl(K)])
        Ljj = L[sl(J), sl(J)]
        if np.any(np.diag(Ljj) == 0.0):
            raise OracleSingular(f"zero diagonal in block {J}")
        X[sl(J)] = la.solve_triangular(Ljj, acc, lower=True,
                                       trans=0 if forward else 1,
                                       check_finite=False)
    return X


def logdet(L, n, bs):
    """bg/distla/kernels.py:493-509: 2 sum log diag over unpadded rows,
    one partial per diagonal block, summed in block order."""
    pn = L.shape[0]
    total = 0.0
    for I in range(1, pn // bs + 1):
        r0 = (I - 1) * bs
        live = min(max(n - r0, 0), bs)
        d = np.diag(L)[r0:r0 + live]
        if np.any(d <= 0.0):
            raise OracleSingular(f"non-positive diagonal in block {I}")
        total += 2.0 * float(np.sum(np.log(d)))
    return total


def sumsq(x, n, bs):
    """bg/distla/kernels.py:512-522."""
    total = 0.0
    for J in range(1, math.ceil(n / bs) + 1):
        lo, hi = (J - 1) * bs, min(J * bs, n)
        total += float(np.dot(x[lo:hi], x[lo:hi]))
    return total


def xprod_mat_vec(V, u, n, m):
    """bg/distla/kernels.py:387-418: w = V^T u (unpadded)."""
    return V[:n, :m].T @ u[:n]


def xprod_self(V, n, m):
    """bg/distla/kernels.py:421-458: tril(V^T V)."""
    return np.tril(V[:n, :m].T @ V[:n, :m])


def xprod_self_diag(V, n, m):
    """bg/distla/kernels.py:461-487: diag(V^T V)."""
    W = V[:n, :m]
    return np.einsum("ij,ij->j", W, W)


# ---------------------------------------------------------------------------
# GP engine (bg/gp/problem.py) at P = 1


class OracleProblem:
    """bg/gp/problem.py:74-300 restated on padded dense arrays (P = 1)."""

    def __init__(self, kernel, coords, y, theta, pred_coords=None, bs=None,
                 bs_m=None, **kernel_inputs):
        self.kernel = kernel
        self.inputs = {"coords": np.asarray(coords, dtype=float)}
        if pred_coords is not None:
            self.inputs["pred_coords"] = np.asarray(pred_coords, dtype=float)
        self.inputs.update(kernel_inputs)
        self.y = np.asarray(y, dtype=float)
        self.n = len(self.y)
        self.m = 0 if pred_coords is None else len(self.inputs["pred_coords"])
        self.theta = np.asarray(theta, dtype=float)
        self.bs = bs or block_size(self.n, default_h(self.n))
        self.bs_m = bs_m or (block_size(self.m, default_h(self.m)) if self.m else 1)
        g = lambda part: Generator(f"gen.{kernel}.{part}")
        self.cov, self.cross, self.pred, self.predvar = (
            g("cov"), g("cross"), g("pred"), g("predvar"))

    def factor(self, theta=None):
        """_ensure_chol, bg/gp/problem.py:119-142."""
        theta = self.theta if theta is None else np.asarray(theta, dtype=float)
        C = construct_triangular(self.cov, theta, self.inputs, self.n, self.bs)
        L = cholesky(C, self.bs)
        pn = L.shape[0]
        resid = np.zeros(pn)
        resid[:self.n] = self.y          # mean_fn = gen.zero
        u = solve_vector(L, resid, self.bs, forward=True)
        return L, u

    def log_density(self, theta=None):
        """bg/gp/problem.py:170-183: -n/2 log 2pi - logdet/2 - ssq/2."""
        L, u = self.factor(theta)
        ld = logdet(L, self.n, self.bs)
        ssq = sumsq(u, self.n, self.bs)
        return -0.5 * self.n * LOG_2PI - 0.5 * ld - 0.5 * ssq

    def _basis(self, theta):
        """_ensure_prediction_basis, bg/gp/problem.py:144-167."""
        L, u = self.factor(theta)
        Cx = construct_rectangular(self.cross, theta, self.inputs, self.n,
                                   self.m, self.bs, self.bs_m)
        V = solve_rect(L, Cx, self.bs, forward=True)
        w = xprod_mat_vec(V, u, self.n, self.m)
        return L, u, V, w

    def predict(self, se_fit=False, theta=None):
        """bg/gp/problem.py:221-244 (pred_mean_fn = gen.zero)."""
        theta = self.theta if theta is None else np.asarray(theta, dtype=float)
        _, _, V, w = self._basis(theta)
        mean = w.copy()
        if not se_fit:
            return mean
        prior = construct_vector(self.predvar, theta, self.inputs, self.m,
                                 self.bs_m)[:self.m]
        se2 = prior - xprod_self_diag(V, self.n, self.m)
        se2 = np.maximum(se2, 0.0)
        return mean, np.sqrt(se2)

    def prediction_variance(self, theta=None):
        """bg/gp/problem.py:246-265."""
        theta = self.theta if theta is None else np.asarray(theta, dtype=float)
        _, _, V, _ = self._basis(theta)
        Cp = construct_triangular(self.pred, theta, self.inputs, self.m,
                                  self.bs_m)[:self.m, :self.m]
        lower = Cp - xprod_self(V, self.n, self.m)
        return lower + np.tril(lower, -1).T


# ---------------------------------------------------------------------------
# BASELINE.json input recipes


def config_inputs(config, n=None, seed=0):
    """Seeded synthetic inputs of BASELINE.json configs 1-5.

    Returns (kernel, coords, theta, kernel_inputs, z).  y = L(theta) z is
    produced by the caller with any correct FP64 Cholesky (C4's is frozen in
    tests/golden/).  Coordinates are iid U[0,1]^2; C4 appends 10 % jittered
    duplicates (sigma 1e-4), C5 is squared-exponential + nugget.
    """
    rng = np.random.default_rng(seed)
    if config == 1:
        n = n or 2048
        X = rng.uniform(0, 1, (n, 2))
        return "matern-nugget", X, np.array([1.0, 0.1, 0.01]), {"nu": 0.5}, \
            rng.standard_normal(n)
    if config == 2:
        n = n or 16384
        X = rng.uniform(0, 1, (n, 2))
        return "matern-nugget", X, np.array([2.0, 0.05, 0.05]), {"nu": 1.5}, \
            rng.standard_normal(n)
    if config == 3:
        n = n or 32768
        X = rng.uniform(0, 1, (n, 2))
        return "matern-nugget", X, np.array([1.0, 0.1, 0.01]), {"nu": 0.5}, \
            rng.standard_normal(n)
    if config == 4:
        n = n or 67275
        n_dup = n // 10
        n_base = n - n_dup
        base = rng.uniform(0, 1, (n_base, 2))
        idx = rng.choice(n_base, n_dup, replace=False)
        X = np.concatenate([base, base[idx] + 1e-4 * rng.standard_normal((n_dup, 2))])
        return "matern-nugget", X, np.array([1.0, 0.08, 0.02]), {"nu": 0.5}, \
            rng.standard_normal(n)
    if config == 5:
        n = n or 131072
        X = rng.uniform(0, 1, (n, 2))
        return "sqexp-nugget", X, np.array([1.0, 0.02, 0.1]), {}, \
            rng.standard_normal(n)
    raise ValueError(config)


def c3_pred_coords(m_side=64):
    """C3 prediction grid: 64 x 64 over [0,1]^2, xy meshgrid order."""
    g = np.linspace(0, 1, m_side)
    return np.stack(np.meshgrid(g, g, indexing="xy"), -1).reshape(-1, 2)


def dense_cov(kernel, theta, X, Y=None, nugget=True, **kernel_inputs):
    """Dense covariance with the generator formulas (for y = L z recipes)."""
    X = _points(X)
    Y = X if Y is None else _points(Y)
    gen = Generator(f"gen.{kernel}.{'cov' if nugget else 'cross'}")
    inputs = {"coords": X, "pred_coords": Y}
    inputs.update(kernel_inputs)
    n, m = len(X), len(Y)
    out = np.empty((n, m))
    step = max(1, 4_000_000 // max(m, 1))
    for r0 in range(0, n, step):
        r1 = min(n, r0 + step)
        ii, jj = np.meshgrid(np.arange(r0 + 1, r1 + 1), np.arange(1, m + 1),
                             indexing="ij")
        out[r0:r1] = gen(theta, inputs, ii.ravel(), jj.ravel()).reshape(r1 - r0, m)
    return out
