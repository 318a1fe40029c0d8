"""The five BASELINE.json workloads as seeded synthetic inputs.

BASELINE.json names no public dataset; every input is generated here on the
host in NumPy float64 and handed bit-identically to the GPU path and to the
CPU oracle (the exact-zero emission masks depend on it, SURVEY §7 hard
part 1).  Conventions pinned by SURVEY §8(d):

* grid as `RunConfig.build_grid` (diagsweep/config.py:199-208): interior
  [a, b] with n cells, h = (b-a)/n, extent [a - pml h, b + pml h],
  n + 2 pml + 1 nodes;  partition `make_partition(grid, counts, d, pml)`
  with d = pml width; `PmlProfile(pml, d, 40.0, 2)`;
* sources f = exp(-sum_a (x_a - c_a)^2 / (2 (2h)^2)) over the whole grid
  (axes broadcast in order), complex128, stacked [nRHS, *counts];
* seeds rng_src = default_rng(1000+k), rng_med = default_rng(2000+k);
* heterogeneous media: c = (c_top + slope z/depth)(1 + amp g),
  g = gaussian_filter(standard_normal(interior nodes), sigma, mode="reflect"),
  g /= max|g|; omega = 2 pi min(c) / (8 h).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .ddm import build_global_operator, build_operators
from .grid import make_grid
from .media import constant_model, raster_model
from .partition import make_partition
from .pml import PmlProfile


@dataclass
class Spec:
    name: str
    interior: tuple  # ((a, b), ...)
    cells: tuple
    pml: int
    d: int
    counts: tuple
    omega: float | None  # None: derived from the medium
    nrhs: int
    mode: str  # "direct" | "gmres"
    medium: str  # "constant" | "raster"
    seed: int
    c_range: tuple = (1.0, 1.0)  # raster: (top speed, speed increase over the depth)
    noise: float = 0.0
    filt: float = 0.0
    src_depth_h: float | None = None  # raster: sources at depth = this * h
    centers: tuple | None = None
    sigma_max: float = 40.0
    exponent: int = 2


def spec(k) -> Spec:
    """Config k in {1, 2, 3, 4, 5, '5r'}."""
    if k == 1:
        return Spec("cfg1-2d-const-185^2-4x4", ((0.0, 1.0),) * 2, (160, 160), 12, 12, (4, 4),
                    2 * math.pi * 16, 1, "direct", "constant", 1, centers=((0.3, 0.4),))
    if k == 2:
        return Spec("cfg2-2d-const-433^2-8x8-16rhs", ((0.0, 1.0),) * 2, (400, 400), 16, 16, (8, 8),
                    2 * math.pi * 40, 16, "direct", "constant", 2)
    if k == 3:
        return Spec("cfg3-2d-hetero-1241x441-16x8-64rhs-gmres", ((0.0, 12.0), (0.0, 4.0)),
                    (1200, 400), 20, 20, (16, 8), None, 64, "gmres", "raster", 3,
                    c_range=(1.5, 3.0), noise=0.15, filt=10.0, src_depth_h=5.0)
    if k == 4:
        return Spec("cfg4-3d-const-109^3-4x4x4-8rhs", ((0.0, 1.0),) * 3, (96, 96, 96), 6, 6,
                    (4, 4, 4), 2 * math.pi * 12, 8, "direct", "constant", 4)
    if k == 5:
        return Spec("cfg5-3d-hetero-145^2x113-4x4x4-32rhs-gmres", ((0.0, 1.0), (0.0, 1.0), (0.0, 0.75)),
                    (128, 128, 96), 8, 8, (4, 4, 4), None, 32, "gmres", "raster", 5,
                    c_range=(1.5, 2.5), noise=0.10, filt=6.0, src_depth_h=5.0)
    if k == "5r":
        return Spec("cfg5r-3d-hetero-57^2x45-4x4x4-4rhs-gmres", ((0.0, 1.0), (0.0, 1.0), (0.0, 0.75)),
                    (48, 48, 36), 4, 2, (4, 4, 4), None, 4, "gmres", "raster", 5,
                    c_range=(1.5, 2.5), noise=0.10, filt=6.0 * 48 / 128, src_depth_h=5.0)
    raise ValueError(f"unknown config {k!r}")


def grid_of(s: Spec):
    extents, counts = [], []
    for (a, b), n in zip(s.interior, s.cells):
        h = (b - a) / n
        extents.append((a - s.pml * h, b + s.pml * h))
        counts.append(n + 2 * s.pml + 1)
    return make_grid(extents, counts)


def velocity_samples(s: Spec) -> np.ndarray | None:
    """Raster speed on the interior nodes (float64), or None for constant c=1."""
    if s.medium == "constant":
        return None
    from scipy.ndimage import gaussian_filter

    rng_med = np.random.default_rng(2000 + s.seed)
    nodes = tuple(n + 1 for n in s.cells)
    g = gaussian_filter(rng_med.standard_normal(nodes), sigma=s.filt, mode="reflect")
    g = g / np.max(np.abs(g))
    depth_axis = len(nodes) - 1
    a, b = s.interior[depth_axis]
    z = np.linspace(a, b, nodes[depth_axis])
    shape = [1] * len(nodes)
    shape[depth_axis] = -1
    top, slope = s.c_range
    return (top + slope * z / (b - a)).reshape(shape) * (1.0 + s.noise * g)


def model_of(s: Spec):
    c = velocity_samples(s)
    if c is None:
        return constant_model(1.0), None
    return raster_model(s.interior, c), c


def omega_of(s: Spec, c) -> float:
    if s.omega is not None:
        return s.omega
    h = min((b - a) / n for (a, b), n in zip(s.interior, s.cells))
    return 2 * math.pi * float(np.min(c)) / (8 * h)


def source_centers(s: Spec):
    if s.centers is not None:
        return [tuple(c) for c in s.centers]
    rng_src = np.random.default_rng(1000 + s.seed)
    dim = len(s.cells)
    if s.medium == "constant":
        return [tuple(c) for c in rng_src.uniform(0, 1, (s.nrhs, dim))]
    h = (s.interior[-1][1] - s.interior[-1][0]) / s.cells[-1]
    depth = s.src_depth_h * h
    if dim == 2:
        xs = rng_src.uniform(s.interior[0][0], s.interior[0][1], s.nrhs)
        return [(float(x), depth) for x in xs]
    xy = rng_src.uniform(0, 1, (s.nrhs, 2))
    return [(float(x), float(y), depth) for x, y in xy]


def sources(s: Spec, grid, centers=None) -> np.ndarray:
    """f[r] = exp(-|x - c_r|^2 / (2 (2h)^2)) on the whole grid, complex128."""
    centers = source_centers(s) if centers is None else centers
    h = grid.spacing[0]
    dim = grid.dim
    out = np.empty((len(centers),) + grid.counts, dtype=np.complex128)
    for r, c in enumerate(centers):
        r_sq = np.zeros(grid.counts)
        for a in range(dim):
            shape = [1] * dim
            shape[a] = -1
            r_sq = r_sq + ((grid.axis_coords(a) - c[a]) ** 2).reshape(shape)
        out[r] = np.exp(-r_sq / (2.0 * (2.0 * h) ** 2))
    return out


def build(s: Spec, assembly: str = "host"):
    """(grid, partition, profile, model, omega, operators, global operator, c).
    assembly="device": raster kappa^2 interpolated on the GPU (K8a, bitwise
    equal to the host path)."""
    grid = grid_of(s)
    part = make_partition(grid, s.counts, s.d, s.pml)
    profile = PmlProfile(s.pml, s.d, s.sigma_max, s.exponent)
    model, c = model_of(s)
    omega = omega_of(s, c)
    ops = build_operators(part, profile, model, omega, assembly=assembly)
    gop = build_global_operator(part, profile, model, omega, assembly=assembly)
    return dict(grid=grid, partition=part, profile=profile, model=model, omega=omega, ops=ops,
                gop=gop, c=c)


def oracle_problem(s: Spec, built: dict):
    """Raw parameters for the oracle (`oracle.ds_oracle.Problem`)."""
    grid = built["grid"]
    c = built["c"]
    velocity = ("const", 1.0) if c is None else ("raster", tuple(s.interior), c)
    return dict(extents=grid.extents, counts=grid.counts, part_counts=s.counts, d=s.d,
                pml=s.pml, sigma_max=s.sigma_max, exponent=s.exponent, omega=built["omega"],
                velocity=velocity)
