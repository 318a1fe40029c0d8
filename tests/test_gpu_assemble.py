"""Device assembly (K8) against the host path: raster
kappa^2 of every operator window bitwise equal (configs 3, 5r and a 3D
raster with a one-point axis), Gaussian source batches within a few ulp with
identical exact-zero sets, and a DDM application on device-assembled
operators bitwise equal to the host-assembled one."""
import numpy as np
import pytest

from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve
from paper_2002_05327_b200.assemble import config_sources_device, gaussian_source_device
from paper_2002_05327_b200.errors import ModelError
from paper_2002_05327_b200.media import RasterModel, gaussian_source
from paper_2002_05327_b200.pml import assemble_operator

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [3, "5r", 5])
def test_raster_kappa2_bitwise(cuda, cfg):
    s = configs.spec(cfg)
    hb = configs.build(s)
    db = configs.build(s, assembly="device")
    for idx, op in hb["ops"].items():
        assert op.kappa2_kind == "full"
        assert np.array_equal(op.kappa2, db["ops"][idx].kappa2), idx
        assert op.fingerprint == db["ops"][idx].fingerprint
    assert np.array_equal(hb["gop"].kappa2, db["gop"].kappa2)


def test_raster_kappa2_degenerate_axis_and_model_error(cuda):
    s = configs.spec("5r")
    b = configs.build(s)
    part, prof = b["partition"], b["profile"]
    rng = np.random.default_rng(7)
    flat = RasterModel(((0.0, 1.0), (0.0, 1.0), (0.0, 0.75)),
                       (1.5 + rng.random((9, 1, 5))).astype(np.float32))  # one-point axis
    idx = next(iter(part.subdomains()))
    args = (part.grid, part.window(idx), part.box(idx), prof, flat, b["omega"])
    h = assemble_operator(*args, clamp_box=part.interior_box())
    d = assemble_operator(*args, clamp_box=part.interior_box(), assembly="device")
    assert np.array_equal(h.kappa2, d.kappa2)
    bad = RasterModel(flat.extents, flat.samples.copy())
    object.__setattr__(bad, "samples", -bad.samples)  # bypass the constructor's check
    with pytest.raises(ModelError):
        assemble_operator(*args[:4], bad, args[5], clamp_box=part.interior_box(),
                          assembly="device")


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_sources_device(cuda, cfg):
    s = configs.spec(cfg)
    grid = configs.grid_of(s)
    cen = configs.source_centers(s)[:4]
    host = configs.sources(s, grid, centers=cen)
    dev = config_sources_device(grid, cen).cpu().numpy()
    assert np.array_equal(host == 0, dev == 0)  # exact-zero (underflow) set
    nz = host != 0
    ulp = np.abs(dev[nz].real - host[nz].real) / np.spacing(np.abs(host[nz].real))
    assert ulp.max() <= 4, ulp.max()
    assert np.all(dev.imag == 0)


def test_gaussian_source_device(cuda):
    s = configs.spec(1)
    grid = configs.grid_of(s)
    host = gaussian_source(grid, (0.3, 0.4), 2 * np.pi * 16)
    dev = gaussian_source_device(grid, (0.3, 0.4), 2 * np.pi * 16).cpu().numpy()
    assert np.array_equal(host == 0, dev == 0)
    nz = host != 0
    assert (np.abs(dev[nz] - host[nz]) / np.spacing(np.abs(host[nz].real))).max() <= 4


def test_ddm_on_device_assembled_operators(cuda):
    s = configs.spec("5r")
    hb, db = configs.build(s), configs.build(s, assembly="device")
    f = configs.sources(s, hb["grid"])[:2]
    uh, _ = diagonal_sweep_solve(f, hb["partition"], hb["ops"], FactorizationCache(),
                                 warn_collar=False)
    ud, _ = diagonal_sweep_solve(f, db["partition"], db["ops"], FactorizationCache(),
                                 warn_collar=False)
    assert np.array_equal(uh.values, ud.values)
