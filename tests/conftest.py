"""Shared fixtures: markers, golden fixtures, serial numpy helpers.

`-m "not gpu"` tests run here (no GPU): the oracle against the golden
vectors, host logic, and the C-ABI library load.  `-m gpu` tests call the
CUDA path through the C-ABI and compare with the oracle / goldens.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden_small.npz"))


@pytest.fixture(scope="session")
def golden_scalars():
    with open(os.path.join(GOLDEN, "golden_scalars.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def c4_scalars():
    with open(os.path.join(GOLDEN, "c4_scalars.json")) as f:
        return json.load(f)


def spd_matrix(n, seed=0):
    """A = B B^T + n I (the reference suite's conftest recipe)."""
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((n, n))
    return B @ B.T + n * np.eye(n)


def exp_cov(coords, sigma2, rho, tau2=0.0):
    coords = np.asarray(coords, dtype=float)
    if coords.ndim == 1:
        coords = coords[:, None]
    d = np.sqrt(((coords[:, None, :] - coords[None, :, :]) ** 2).sum(-1))
    return sigma2 * np.exp(-d / rho) + tau2 * np.eye(len(coords))


def relerr(got, want):
    want = np.asarray(want, dtype=float)
    scale = np.linalg.norm(want)
    return np.linalg.norm(np.asarray(got) - want) / (scale if scale else 1.0)


@pytest.fixture
def cluster_factory():
    """GPU clusters, shut down at test end."""
    from paper_1305_4886_b200 import spawn
    opened = []

    def make(P=1, **kwargs):
        cl = spawn(P, **kwargs)
        opened.append(cl)
        return cl

    yield make
    for cl in opened:
        cl.shutdown()
