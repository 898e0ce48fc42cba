"""B200-native bigGP likelihood path: a drop-in for the `blockgp` API.

Covariance construction, tiled Cholesky, triangular solves, log-density and
kriging predict / variance run as hand-written sm_100a CUDA kernels
(libbgp.so, include/bgp.h); this package is the host-side mirror of the
reference's Python interface (`spawn`, `distla`, `gp.KrigeProblem`,
`errors`).  Importing it registers every device operation and generator.
"""

from . import distla, gp  # noqa: F401  (register device ops and generators)
from .errors import *  # noqa: F401,F403
from .grid import BlockLayout, DeviceGrid, ProcessGrid, default_h, grid_from_process_count
from .transport import spawn

__version__ = "0.1.0"
