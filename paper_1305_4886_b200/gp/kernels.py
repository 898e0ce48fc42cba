"""Covariance kernels: host correlation functions (public API) and the
device generator ids behind `builtin_spec`.

`matern_correlation` / `sqexp_correlation` are the scalar/array utilities of
bg/gp/kernels.py:16-34 (used by callers for checks and plotting); they never
run on the likelihood path.  The generator ids registered here
(bg/gp/kernels.py:49-180) are bound to the device kernel K1
(csrc/cov.cu) through `registry.DeviceGenerator`.
"""

import numpy as np

from .. import registry
from .._lib import (GEN_DELTA, GEN_LINEAR_INDEX, GEN_MATERN, GEN_PRODUCT,
                    GEN_SQEXP, GEN_WHITE, GEN_ZERO, PART_COV, PART_CROSS,
                    PART_PRED, PART_PREDVAR)
from ..errors import UnsupportedSmoothness

HALF_INTEGER_NU = (0.5, 1.5, 2.5)


def matern_correlation(d, rho, nu):
    """Half-integer Matern correlation, s = sqrt(2 nu) d / rho."""
    d = np.asarray(d, dtype=float)
    if rho <= 0:
        raise ValueError(f"range must be positive, got {rho}")
    if nu not in HALF_INTEGER_NU:
        raise UnsupportedSmoothness(f"nu={nu} not supported; use one of {HALF_INTEGER_NU}")
    s = np.sqrt(2.0 * nu) * d / rho
    poly = {0.5: 1.0, 1.5: 1.0 + s, 2.5: 1.0 + s + s * s / 3.0}[nu]
    return poly * np.exp(-s)


def sqexp_correlation(d, rho):
    """Squared-exponential correlation exp(-(d/rho)^2 / 2)."""
    d = np.asarray(d, dtype=float)
    return np.exp(-0.5 * (d / rho) ** 2)


def make_pairwise(kernel_id, corr):
    """Register gen.<kernel_id>.{cov,cross,pred,predvar} on a device kernel.

    `corr` is "matern" or "sqexp"; theta[0] is the marginal variance and a
    kernel id ending in "-nugget" adds theta[-1] on the observation
    diagonal only (same contract as bg/gp/kernels.py:68-98).
    """
    family = {"matern": GEN_MATERN, "sqexp": GEN_SQEXP}[corr]
    nugget = kernel_id.endswith("-nugget")
    for part, code in (("cov", PART_COV), ("cross", PART_CROSS),
                       ("pred", PART_PRED), ("predvar", PART_PREDVAR)):
        registry.register(f"gen.{kernel_id}.{part}",
                          registry.DeviceGenerator(family, code, nugget and part == "cov", corr))


registry.register("gen.zero", registry.DeviceGenerator(GEN_ZERO, PART_COV, False))
registry.register("gen.delta", registry.DeviceGenerator(GEN_DELTA, PART_COV, False))
registry.register("gen.linear_index", registry.DeviceGenerator(GEN_LINEAR_INDEX, PART_COV, False))

make_pairwise("sqexp", "sqexp")                    # theta = (sigma2, rho)
make_pairwise("matern", "matern")                  # theta = (sigma2, rho)
make_pairwise("matern-nugget", "matern")           # theta = (sigma2, rho, tau2)
# BASELINE config 5 (squared exponential + nugget); registered through the
# same extension point the reference offers (not a reference built-in)
make_pairwise("sqexp-nugget", "sqexp")             # theta = (sigma2, rho, tau2)

for _part, _code in (("cov", PART_COV), ("cross", PART_CROSS), ("pred", PART_PRED),
                     ("predvar", PART_PREDVAR)):
    registry.register(f"gen.matern-product-nugget.{_part}",
                      registry.DeviceGenerator(GEN_PRODUCT, _code, _part == "cov", "matern"))
    registry.register(f"gen.white.{_part}",
                      registry.DeviceGenerator(GEN_WHITE, _code, False))

BUILTIN_KERNELS = {
    "sqexp": 2,
    "matern": 2,
    "matern-nugget": 3,
    "matern-product-nugget": 4,
    "white": 1,
}
