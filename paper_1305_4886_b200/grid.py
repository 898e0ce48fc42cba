"""Layout metadata of the drop-in API and the GPU tile ownership map.

`BlockLayout` and `default_h` keep the reference semantics exactly
(bg/grid.py:77-113): a dimension of n points cut into B = h*D blocks of
ceil(n/B) with identity / zero padding to B*block_size.  They describe the
API-level blocking (what `NotPositiveDefinite.block_index` counts in); the
device stores every object in its own b x b tiles (include/bgp.h), so any
layout works with any tile size.

The reference's triangular D(D+1)/2 process fold (bg/grid.py:116-139) is
replaced by `DeviceGrid`: G GPUs in a Pr x Pc grid owning lower tiles
2-D block-cyclically, owner(I, J) = (I mod Pr, J mod Pc).
"""

from dataclasses import dataclass
from math import ceil, isqrt

from .errors import DimensionMismatch, NotTriangularNumber, OutOfTriangle

DEFAULT_BLOCK_TARGET = 1000


@dataclass(frozen=True)
class BlockLayout:
    """API blocking of 1..n into B = h*D blocks (bg/grid.py:77-105)."""

    n: int
    h: int
    D: int

    def __post_init__(self):
        if self.n < 1 or self.h < 1 or self.D < 1:
            raise DimensionMismatch(f"invalid layout n={self.n} h={self.h} D={self.D}")

    @property
    def B(self):
        return self.h * self.D

    @property
    def block_size(self):
        return ceil(self.n / self.B)

    @property
    def padded_n(self):
        return self.B * self.block_size

    def block_range(self, J):
        """1-based inclusive global index range of block J (padded)."""
        bs = self.block_size
        return (J - 1) * bs + 1, J * bs


def default_h(n, D, target=DEFAULT_BLOCK_TARGET):
    """Smallest h with ceil(n/(h*D)) <= target (bg/grid.py:108-113)."""
    h = max(1, ceil(n / (target * D)))
    while h > 1 and ceil(n / ((h - 1) * D)) <= target:
        h -= 1
    while ceil(n / (h * D)) > target:
        h += 1
    return h


def triangular_order(P):
    if P < 1:
        raise NotTriangularNumber(f"P must be >= 1, got {P}")
    D = (isqrt(8 * P + 1) - 1) // 2
    if D * (D + 1) // 2 != P:
        raise NotTriangularNumber(f"{P} is not a triangular number")
    return D


@dataclass(frozen=True)
class ProcessGrid:
    """The reference's triangular worker grid (kept for API compatibility;
    the b200 runtime uses DeviceGrid)."""

    D: int

    @property
    def P(self):
        return self.D * (self.D + 1) // 2

    def coord_to_rank(self, y, z):
        if not (1 <= z <= y <= self.D):
            raise OutOfTriangle(f"({y},{z}) not in lower triangle of order {self.D}")
        return (z - 1) * self.D - (z - 1) * (z - 2) // 2 + (y - z + 1)

    def rank_to_coord(self, rank):
        if not (1 <= rank <= self.P):
            raise OutOfTriangle(f"rank {rank} outside 1..{self.P}")
        z, r = 1, rank
        while r > self.D - z + 1:
            r -= self.D - z + 1
            z += 1
        return (z + r - 1, z)


def grid_from_process_count(P):
    return ProcessGrid(triangular_order(P))


def block_owner(I, J, grid):
    """Reference-layout owner coordinate of lower block (I, J): both indices
    folded to their residue in 1..D and sorted (bg/grid.py:116-139).  Kept so
    layout queries of reference code resolve; the device uses DeviceGrid."""
    if J > I:
        raise OutOfTriangle(f"block ({I},{J}) above the diagonal")
    a, c = (I - 1) % grid.D + 1, (J - 1) % grid.D + 1
    return (max(a, c), min(a, c))


def triangular_blocks(coord, layout, grid):
    """Reference-layout lower blocks held by worker `coord`, column-major."""
    return [(I, J) for J in range(1, layout.B + 1) for I in range(J, layout.B + 1)
            if block_owner(I, J, grid) == tuple(coord)]


def _grid_shape(G):
    """Pr x Pc with Pr <= Pc, Pr*Pc = G, as square as possible (1x1, 1x2, 2x2, 2x4)."""
    pr = isqrt(G)
    while G % pr:
        pr -= 1
    return pr, G // pr


@dataclass(frozen=True)
class DeviceGrid:
    """G GPUs as a Pr x Pc grid; lower tile (I, J) (0-based) lives on
    rank (I mod Pr) + Pr * (J mod Pc) (0-based rank)."""

    G: int

    def __post_init__(self):
        if self.G < 1:
            raise DimensionMismatch(f"device count must be >= 1, got {self.G}")

    @property
    def P(self):
        return self.G

    @property
    def D(self):
        # API layouts on the device grid are independent of the process
        # count: one "process dimension"
        return 1

    @property
    def shape(self):
        return _grid_shape(self.G)

    def owner(self, I, J):
        pr, pc = self.shape
        return (I % pr) + pr * (J % pc)

    def owned_tiles(self, rank, T):
        """Lower tiles (I, J), I >= J, owned by `rank`, column-major."""
        return [(I, J) for J in range(T) for I in range(J, T) if self.owner(I, J) == rank]

    def rank_to_coord(self, rank):
        pr, _ = self.shape
        r = rank - 1
        return (r % pr + 1, r // pr + 1)

    def coord_to_rank(self, y, z):
        pr, _ = self.shape
        return (y - 1) + pr * (z - 1) + 1
