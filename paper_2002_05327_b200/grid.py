"""Node-centred tensor grids, inclusive index windows and complex fields.

Host metadata only (nothing here touches the GPU).  Semantics follow
`diagsweep/grid.py`: `Grid` (`grid.py:20-43`, spacing = extent/(n-1), nodes
from `np.linspace`), `Window` inclusive boxes (`grid.py:46-79`) and
`make_grid` validation (`grid.py:99-109`).  `ComplexField` additionally
accepts a leading right-hand-side batch axis, since the GPU engine works on
`[nrhs, *grid.counts]` batches.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError


@dataclass(frozen=True)
class Grid:
    extents: tuple[tuple[float, float], ...]
    counts: tuple[int, ...]

    @property
    def dim(self) -> int:
        return len(self.counts)

    @property
    def spacing(self) -> tuple[float, ...]:
        return tuple((hi - lo) / (n - 1) for (lo, hi), n in zip(self.extents, self.counts))

    def axis_coords(self, axis: int) -> np.ndarray:
        lo, hi = self.extents[axis]
        return np.linspace(lo, hi, self.counts[axis])

    def node_count(self) -> int:
        return math.prod(self.counts)

    def full_window(self) -> "Window":
        return Window((0,) * self.dim, tuple(n - 1 for n in self.counts))


@dataclass(frozen=True)
class Window:
    """Inclusive node-index box [lo, hi]."""

    lo: tuple[int, ...]
    hi: tuple[int, ...]

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(b - a + 1 for a, b in zip(self.lo, self.hi))

    @property
    def size(self) -> int:
        return math.prod(self.shape)

    def slices(self) -> tuple[slice, ...]:
        return tuple(slice(a, b + 1) for a, b in zip(self.lo, self.hi))

    def contains(self, node) -> bool:
        return all(a <= p <= b for p, a, b in zip(node, self.lo, self.hi))

    def intersect(self, other: "Window") -> "Window | None":
        lo = tuple(map(max, self.lo, other.lo))
        hi = tuple(map(min, self.hi, other.hi))
        if any(a > b for a, b in zip(lo, hi)):
            return None
        return Window(lo, hi)

    def local_slices(self, sub: "Window") -> tuple[slice, ...]:
        return tuple(slice(s - a, t - a + 1) for a, s, t in zip(self.lo, sub.lo, sub.hi))

    def grow(self, points: int) -> "Window":
        return Window(tuple(a - points for a in self.lo), tuple(b + points for b in self.hi))


class ComplexField:
    """Complex nodal values on a grid: `[*counts]` or batched `[nrhs, *counts]`.

    `values` may be a NumPy array or a torch tensor (device-resident results
    of the GPU engine stay on the device unless the caller asks for NumPy).
    """

    def __init__(self, grid: Grid, values):
        shape = tuple(values.shape)
        if shape != grid.counts and shape[1:] != grid.counts:
            raise ConfigurationError(
                f"field shape {shape} does not match grid {grid.counts}"
            )
        self.grid = grid
        self.values = values

    @property
    def batched(self) -> bool:
        return tuple(self.values.shape) != self.grid.counts

    def numpy(self) -> np.ndarray:
        v = self.values
        if hasattr(v, "detach"):
            v = v.detach().cpu().numpy()
        return np.asarray(v)

    def copy(self) -> "ComplexField":
        return ComplexField(self.grid, self.values.copy() if isinstance(self.values, np.ndarray)
                            else self.values.clone())


def make_grid(extents, counts) -> Grid:
    extents = tuple((float(a), float(b)) for a, b in extents)
    counts = tuple(int(n) for n in counts)
    if len(extents) != len(counts) or len(counts) not in (2, 3):
        raise ConfigurationError("grid must be 2D or 3D with matching extents/counts")
    for (a, b), n in zip(extents, counts):
        if n < 2:
            raise ConfigurationError(f"axis needs at least 2 points, got {n}")
        if not b > a:
            raise ConfigurationError(f"degenerate extent [{a}, {b}]")
    return Grid(extents, counts)
