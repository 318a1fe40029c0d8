"""Source-transfer geometry and the sweep-admissibility rule engine.

Host-side integer/float64 tables consumed by the GPU transfer kernel (K4):

* `transfer_geometry` restates the band / ext / weight / sign bookkeeping of
  `psi` (`diagsweep/transfer.py:100-155`): band = d+1 layers from the shared
  breakpoint on every nonzero axis (window intersection on zero axes),
  ext = grow(band, 1) ∩ src_win ∩ nb_win, weight = prod_{c!=0} (1 - beta_1d),
  sign = +1 for odd |dir|_1 else -1.
* `similar_direction`, `rule_allows`, `next_usable_sweep`
  (`transfer.py:63-97`) — routing must match the golden tables
  `pkg/tests/data/rule_table_{2d,3d}.csv` bit-exactly.

The payload arithmetic of `psi` runs only inside the sweep engine's fused
transfer kernel (K4, csrc/ds_sweep.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import Window


@dataclass
class TransferredSource:
    target: tuple
    direction: tuple
    gen_sweep: int
    window: Window
    values: object
    cuts: frozenset = frozenset()


def similar_direction(d1, d2, dim: int) -> bool:
    dot = sum(a * b for a, b in zip(d1, d2))
    if dim == 2:
        return dot > 0
    return dot > 0 and not any(a * b < 0 for a, b in zip(d1, d2))


def _coordinate_planes(dim: int):
    return ((0, 1),) if dim == 2 else ((0, 1), (0, 2), (1, 2))


def rule_allows(src_dir, gen_sweep_dir, use_sweep_dir, dim: int) -> bool:
    if not similar_direction(src_dir, use_sweep_dir, dim):
        return False
    for plane in _coordinate_planes(dim):
        zeros = sum(1 for a in plane if src_dir[a] == 0)
        opposite = all(gen_sweep_dir[a] == -use_sweep_dir[a] for a in plane)
        if zeros == 1 and opposite:
            return False
    return True


def next_usable_sweep(src_dir, gen_sweep: int, directions):
    dim = len(src_dir)
    gen_dir = directions[gen_sweep - 1]
    for use in range(gen_sweep, len(directions) + 1):
        if rule_allows(src_dir, gen_dir, directions[use - 1], dim):
            return use
    return None


@dataclass(frozen=True)
class TransferGeometry:
    source: tuple
    target: tuple
    direction: tuple
    band: Window
    ext: Window
    sign: float
    # per-axis (1 - beta_1d) factors on ext (ones on zero axes), float64
    factors: tuple


def transfer_geometry(partition, index, direction) -> TransferGeometry | None:
    target = tuple(i + c for i, c in zip(index, direction))
    if any(not 1 <= t <= n for t, n in zip(target, partition.counts)):
        return None
    d = partition.overlap_d_points
    src_win = partition.window(index)
    nb_win = partition.window(target)
    lo, hi = [], []
    for a, c in enumerate(direction):
        bk = partition.breaks[a]
        i = index[a]
        if c == 1:
            lo.append(bk[i]); hi.append(bk[i] + d)
        elif c == -1:
            lo.append(bk[i - 1] - d); hi.append(bk[i - 1])
        else:
            lo.append(max(src_win.lo[a], nb_win.lo[a])); hi.append(min(src_win.hi[a], nb_win.hi[a]))
    band = Window(tuple(lo), tuple(hi))
    ext = band.grow(1).intersect(src_win).intersect(nb_win)
    factors = []
    for a, c in enumerate(direction):
        nodes = np.arange(ext.lo[a], ext.hi[a] + 1)
        if c == 0:
            factors.append(np.ones(nodes.size))
        else:
            factors.append(1.0 - partition.beta_1d_nodes(a, c, index[a], nodes))
    order = sum(1 for c in direction if c)
    return TransferGeometry(tuple(index), target, tuple(direction), band, ext,
                            1.0 if order % 2 == 1 else -1.0, tuple(factors))


def transfer_weight(geom: TransferGeometry) -> np.ndarray:
    """prod_a (1 - beta_a) on ext, multiplied in axis order like `psi`."""
    dim = len(geom.direction)
    weight = np.ones(geom.ext.shape)
    for a, c in enumerate(geom.direction):
        if c == 0:
            continue
        shape = [1] * dim
        shape[a] = -1
        weight = weight * geom.factors[a].reshape(shape)
    return weight
