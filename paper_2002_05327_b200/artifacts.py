"""File artifacts of the drivers, byte-compatible with the reference.

* fields: raw little-endian float64, (re, im) interleaved, axis 0 fastest,
  plus a JSON sidecar (dims, extents, counts, layout) -- grid.py:163-191;
* quicklook: binary PGM of the real part scaled to [0, 255], rows along
  axis 1 with the largest coordinate on top, 3D fields by their middle slice
  along the last axis -- grid.py:194-209;
* velocity rasters: raw little-endian float32, axis 0 fastest, plus a JSON
  sidecar -- media.py:115-144.

A batched field ([R, *counts]) is written one file per RHS by the CLI; these
functions take one field.  Host code (files are host I/O); tests pin the
bytes against files the reference wrote (tests/test_drivers.py).
"""

from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np

from .errors import ModelError
from .grid import ComplexField, make_grid
from .media import RasterModel


def _sidecar(path: Path) -> Path:
    return path.with_suffix(path.suffix + ".json")


def _host_values(u) -> np.ndarray:
    vals = u.values if isinstance(u, ComplexField) else u
    if hasattr(vals, "detach"):
        vals = vals.detach().cpu().numpy()
    return np.asarray(vals)


def dump_field(u: ComplexField, path) -> None:
    path = Path(path)
    vals = _host_values(u)
    col = vals.ravel(order="F")
    raw = np.empty((col.size, 2), dtype="<f8")
    raw[:, 0] = col.real
    raw[:, 1] = col.imag
    raw.tofile(path)
    g = u.grid
    _sidecar(path).write_text(json.dumps({
        "dims": g.dim, "extents": [list(e) for e in g.extents], "counts": list(g.counts),
        "layout": "f64le re/im interleaved, x fastest"}, indent=2))


def load_field(path) -> ComplexField:
    path = Path(path)
    meta = json.loads(_sidecar(path).read_text())
    grid = make_grid(meta["extents"], meta["counts"])
    pairs = np.fromfile(path, dtype="<f8").reshape(-1, 2)
    vals = (pairs[:, 0] + 1j * pairs[:, 1]).reshape(grid.counts, order="F")
    return ComplexField(grid, np.ascontiguousarray(vals))


def write_pgm(u: ComplexField, path) -> None:
    re = _host_values(u).real
    if re.ndim == 3:
        re = re[:, :, re.shape[2] // 2]
    lo, hi = float(re.min()), float(re.max())
    gain = 255.0 / (hi - lo) if hi > lo else 0.0
    pix = ((re - lo) * gain).astype(np.uint8).T[::-1]
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n255\n" % (pix.shape[1], pix.shape[0]))
        fh.write(pix.tobytes())


def save_velocity(model: RasterModel, path) -> None:
    path = Path(path)
    model.samples.astype("<f4").ravel(order="F").tofile(path)
    _sidecar(path).write_text(json.dumps({
        "counts": list(model.samples.shape), "extents": [list(e) for e in model.extents],
        "dtype": "f32le"}, indent=2))


def load_velocity(path) -> RasterModel:
    path = Path(path)
    side = _sidecar(path)
    if not (path.exists() and side.exists()):
        raise ModelError(f"missing raster file or sidecar for {path}")
    meta = json.loads(side.read_text())
    try:
        counts = tuple(int(n) for n in meta["counts"])
        extents = tuple((float(a), float(b)) for a, b in meta["extents"])
        dtype = meta["dtype"]
    except (KeyError, TypeError, ValueError) as exc:
        raise ModelError(f"malformed raster sidecar {side}: {exc}") from exc
    if dtype != "f32le":
        raise ModelError(f"unsupported raster dtype {dtype!r}")
    raw = np.fromfile(path, dtype="<f4")
    if raw.size != math.prod(counts):
        raise ModelError(f"raster size {raw.size} does not match sidecar counts {counts}")
    return RasterModel(extents, np.ascontiguousarray(raw.reshape(counts, order="F")))
