"""Problem assembly on the device (K8, csrc/ds_assemble.cu).

* `raster_kappa2_device` -- kappa^2 = (omega / c)^2 of an operator window for
  a raster medium (reference pml.py:197-213 `_kappa2_structure`, "full" kind,
  with `RasterModel.speed_at`, media.py:75-101).  The per-axis parts (the
  clamped coordinates, t, the lower raster index and its fraction) are 1D
  NumPy tables computed by the reference's own expressions; K8a does the
  per-node interpolation with explicitly rounded arithmetic in the
  reference's corner order: bitwise the host values.
* `gaussian_fields_device` -- batches of Gaussian sources on the device
  (`configs.sources`: exp(-|x - c|^2 / (2 (2h)^2)); `gaussian_source`,
  media.py:147-167: amp exp(-rate |x - c|^2)), RHS-outer complex128.  The
  squared distances are exact; the exponential is CUDA's (~1 ulp), so values
  agree with NumPy to a few ulp and the exact-zero (underflow) set is equal
  (tests/test_gpu_assemble.py).

`assemble_operator(..., assembly="device")` / `build_operators(...,
assembly="device")` route the raster kappa^2 through K8a; the host keeps a
copy (fingerprints hash its bytes, pml.py:175-186).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .errors import ConfigurationError, ModelError


_RASTER_DEV = None


def _ptr_array(tensors):
    return (C.c_void_p * 3)(*([t.data_ptr() for t in tensors] + [0] * (3 - len(tensors))))


def raster_axis_tables(coords, extent, n):
    """(lower raster index int32, fraction float64) of window coordinates
    along one raster axis -- RasterModel.speed_at's per-axis step."""
    a, b = extent
    t = np.clip((np.asarray(coords, dtype=np.float64) - a) / (b - a) * (n - 1), 0.0, n - 1.0)
    base = np.minimum(t.astype(np.int64), n - 2) if n > 1 else np.zeros_like(t, np.int64)
    return base.astype(np.int32), t - base


def raster_kappa2_device(grid, window, model, omega: float, clamp_box):
    """kappa^2 over `window` for a RasterModel, on the current CUDA device
    (torch float64 tensor of window.shape)."""
    import torch

    from . import _engine

    lib, ctx = _engine.context()
    dim = grid.dim
    samples = np.asarray(model.samples)
    if samples.ndim != dim:
        raise ConfigurationError("raster dimension does not match the grid")
    sl = window.slices()
    bases, fracs = [], []
    for ax in range(dim):
        x = np.clip(grid.axis_coords(ax)[sl[ax]], clamp_box[ax][0], clamp_box[ax][1])
        bi, fr = raster_axis_tables(x, model.extents[ax], samples.shape[ax])
        bases.append(torch.from_numpy(bi).cuda())
        fracs.append(torch.from_numpy(np.ascontiguousarray(fr)).cuda())
    global _RASTER_DEV  # the last raster's samples on the device (one model at a time)
    dev = _RASTER_DEV
    if dev is None or dev[0] is not model:
        dev = _RASTER_DEV = (model, torch.from_numpy(
            np.ascontiguousarray(samples, dtype=np.float64)).cuda())
    out = torch.empty(tuple(window.shape), dtype=torch.float64, device="cuda")
    wc, _ = N.i32_array(window.shape)
    rc, _ = N.i32_array(samples.shape)
    N.check(lib.ds_raster_kappa2(ctx, dim, wc.ctypes.data, rc.ctypes.data, dev[1].data_ptr(),
                                 _ptr_array(bases), _ptr_array(fracs), float(omega),
                                 out.data_ptr()), "ds_raster_kappa2")
    return out


def _distance_tables(grid, centers):
    """Per axis [R, n_a] squared distances (coords - c)**2, as NumPy forms them."""
    import torch

    tabs = []
    for ax in range(grid.dim):
        x = grid.axis_coords(ax)
        d2 = np.stack([(x - float(c[ax])) ** 2 for c in centers])
        tabs.append(torch.from_numpy(np.ascontiguousarray(d2)).cuda())
    return tabs


def gaussian_fields_device(grid, centers, amp=1.0, scale=None, divide=False):
    """[R, *counts] complex128 on the device: amp_r exp(scale_r r2) or, with
    divide=True, amp_r exp(-r2 / scale_r)."""
    import torch

    from . import _engine

    lib, ctx = _engine.context()
    R = len(centers)
    out = torch.empty((R,) + tuple(grid.counts), dtype=torch.complex128, device="cuda")
    if R == 0:
        return out
    tabs = _distance_tables(grid, centers)
    ampv = torch.tensor(np.broadcast_to(np.asarray(amp, np.float64), (R,)).copy(), device="cuda")
    scv = torch.tensor(np.broadcast_to(np.asarray(scale, np.float64), (R,)).copy(), device="cuda")
    cnt, _ = N.i32_array(grid.counts)
    N.check(lib.ds_gaussian_fields(ctx, grid.dim, cnt.ctypes.data, R, _ptr_array(tabs),
                                   ampv.data_ptr(), scv.data_ptr(), int(bool(divide)),
                                   out.data_ptr()), "ds_gaussian_fields")
    return out


def config_sources_device(grid, centers):
    """`configs.sources` on the device: exp(-r2 / (2 (2h)^2)) per center."""
    h = grid.spacing[0]
    return gaussian_fields_device(grid, centers, 1.0, 2.0 * (2.0 * h) ** 2, divide=True)


def gaussian_source_device(grid, center, kappa: float, interior=None):
    """`media.gaussian_source` on the device (one field, complex128)."""
    from .media import _check_inside

    center = tuple(float(c) for c in center)
    _check_inside(center, grid, interior)
    amp = 16.0 * kappa ** 2 / math.pi ** 3 if grid.dim == 2 else 64.0 * kappa ** 3 / math.pi ** 4.5
    rate = (4.0 * kappa / math.pi) ** 2
    return gaussian_fields_device(grid, [center], amp, -rate)[0]


__all__ = ["config_sources_device", "gaussian_fields_device", "gaussian_source_device",
           "raster_axis_tables", "raster_kappa2_device", "ModelError"]
