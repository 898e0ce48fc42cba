"""Handles (master side) and device-resident objects (device store).

The handle types keep the reference's shape (bg/distla/objects.py:31-49):
frozen (name, layout) records the caller passes back into distla calls.
`DevObj` replaces the reference's per-worker `LocalPiece` dict of numpy
blocks: one FP64 torch buffer on the GPU in the packed-tile format of
include/bgp.h, plus its API layouts.
"""

from dataclasses import dataclass
from typing import Any, Optional

from ..grid import BlockLayout


@dataclass(frozen=True)
class DistTriangular:
    """Handle to a lower-triangular distributed matrix."""

    name: str
    layout: BlockLayout


@dataclass(frozen=True)
class DistRectangular:
    name: str
    row_layout: BlockLayout
    col_layout: BlockLayout


@dataclass(frozen=True)
class DistVector:
    name: str
    layout: BlockLayout


@dataclass
class DevObj:
    """One object in the device store.

    kind "triangular": data (T(T+1)/2, b, b) packed lower tiles (tile (I, J)
    at J*T - J(J-1)/2 + I - J, each tile column-major);
    "rectangular" (n x m): data (Tn*Tm, b, b) tiles of the TRANSPOSE (m x n),
    tile (A, I) at I*Tm + A; "vector": data (T*b,) zero padded.
    """

    kind: str
    row_layout: BlockLayout
    col_layout: Optional[BlockLayout]
    tile: int
    data: Any
    dist: Any = None   # parallel.TileDist when the tiles are spread over G > 1 GPUs

    @property
    def n(self):
        return self.row_layout.n

    @property
    def m(self):
        return (self.col_layout or self.row_layout).n


# reference-compatible name for the per-worker piece type
LocalPiece = DevObj
