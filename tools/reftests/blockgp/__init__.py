"""Test-only alias: `import blockgp` resolves to this repo's package.

Lets the reference's OWN test files (pkg/tests/test_distla.py, test_gp.py,
test_acceptance.py; copied at run time by tools/run_reference_tests.sh into
the git-ignored baseline/_ref/tests, never committed) run against the b200
backend unchanged.  Every `blockgp.<mod>` import is served by
`paper_1305_4886_b200.<mod>`; `spawn(P, backend=...)` maps the reference's
triangular worker counts onto GPUs (P in {1, 3, 6, 10} ->
G in {1, 2, 4, 8}) -- by default all on one GPU process (G = 1), or, with
BGP_REFTEST_MULTI=1, G worker processes sharing the available GPUs
(transport.master).  The backend string is ignored (there is only b200).
"""

import importlib
import importlib.abc
import importlib.util
import os
import sys

import paper_1305_4886_b200 as _pkg
from paper_1305_4886_b200 import *  # noqa: F401,F403
from paper_1305_4886_b200 import distla, errors, gp, grid, registry  # noqa: F401
from paper_1305_4886_b200 import spawn as _spawn

_G_OF_P = {1: 1, 3: 2, 6: 4, 10: 8}


def spawn(P=1, backend="b200", seed=0, blas_threads=None, **kwargs):
    G = _G_OF_P.get(P, 1) if os.environ.get("BGP_REFTEST_MULTI") == "1" else 1
    if G > 1:
        import torch
        kwargs.setdefault("devices", [r % torch.cuda.device_count() for r in range(G)])
    kwargs.setdefault("tile", int(os.environ.get("BGP_REFTEST_TILE", "128")))
    return _spawn(G, backend="b200", seed=seed, **kwargs)


class _Alias(importlib.abc.MetaPathFinder, importlib.abc.Loader):
    def find_spec(self, name, path, target=None):
        if name.startswith("blockgp."):
            real = "paper_1305_4886_b200." + name[len("blockgp."):]
            if importlib.util.find_spec(real) is not None:
                return importlib.util.spec_from_loader(name, self)
        return None

    def create_module(self, spec):
        return importlib.import_module("paper_1305_4886_b200." + spec.name[len("blockgp."):])

    def exec_module(self, module):
        pass


sys.meta_path.insert(0, _Alias())
__path__ = []  # a package, so `blockgp.x` imports go through the finder
__version__ = _pkg.__version__
