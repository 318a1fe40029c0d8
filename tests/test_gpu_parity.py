"""CUDA path vs the CPU oracle on the same seeded inputs (parity proper).

Tolerances (SURVEY §8 / BASELINE.json north star): relative L2 <= 1e-10 for
solutions in complex128 -- DDM applications and GMRES solutions alike
(measured on the B200: GMRES x within 1e-15 of the oracle, u_DDM within
1e-12) -- GMRES iteration counts within +-1 (we require equality), counters /
emission events / index maps exact.
"""

import math
import os
from pathlib import Path

import numpy as np
import pytest

from oracle import ds_oracle as O
from paper_2002_05327_b200 import (
    FactorizationCache,
    PmlProfile,
    build_global_operator,
    build_operators,
    configs,
    constant_model,
    diagonal_sweep_solve,
    gaussian_source,
    gmres,
    gmres_batched,
    make_grid,
    make_partition,
    tuned_sigma_max,
)
from paper_2002_05327_b200.grid import Window

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def cfg1():
    s = configs.spec(1)
    b = configs.build(s)
    prob = O.Problem(**configs.oracle_problem(s, b))
    return s, b, prob, prob.operators()


def mini_raster_spec(nrhs=3):
    return configs.Spec("mini-raster", ((0.0, 2.4), (0.0, 0.8)), (240, 80), 10, 10, (4, 2),
                        None, nrhs, "gmres", "raster", 3, c_range=(1.5, 3.0), noise=0.15,
                        filt=10.0, src_depth_h=5.0)


@pytest.fixture(scope="module")
def raster():
    s = mini_raster_spec()
    b = configs.build(s)
    prob = O.Problem(**configs.oracle_problem(s, b))
    return s, b, prob, prob.operators()


def test_stencil_apply_global_and_region(cuda, cfg1):
    s, b, prob, oops = cfg1
    rng = np.random.default_rng(5)
    gop = b["gop"]
    v = rng.standard_normal((3,) + gop.window.shape) + 1j * rng.standard_normal((3,) + gop.window.shape)
    out = gop.apply(v)
    ogop = prob.global_operator()
    for r in range(3):
        assert rel(out[r], ogop.apply(v[r])) <= 1e-14
    # sub-region with zero outside (pml.py:135-159)
    op = b["ops"][(2, 3)]
    w = op.window
    reg = Window(tuple(l + 3 for l in w.lo), tuple(l + 20 for l in w.lo))
    vr = rng.standard_normal(reg.shape) + 1j * rng.standard_normal(reg.shape)
    got = op.apply(vr, region=reg)
    want = oops[(2, 3)].apply(vr, reg.lo)
    assert rel(got, want) <= 1e-14


@pytest.mark.parametrize("k1", [4, 8, 2, 16, 0])
def test_stencil_variants_ragged_regions(cuda, k1):
    """K1 variants (column marching with 4 / 8 / 2 / 16 rows per thread, 0 =
    the 32 x 8 shared-memory tile; context option "k1", switched in-process)
    on ragged regions (strip edges, warp edges, last row block partial) and
    several RHS planes: <= 1e-14 vs the oracle, and bitwise equal to each
    other."""
    from paper_2002_05327_b200 import _engine

    old = _engine.set_option("k1", k1)
    try:
        got = _ragged_stencil_case()
    finally:
        _engine.set_option("k1", old)
    ref = _RAGGED_REF.setdefault("u", got)
    assert np.array_equal(got, ref), k1


_RAGGED_REF: dict = {}


def _ragged_stencil_case():
    """Run in a child process: the global config-1 operator applied to 5 RHS
    over three ragged regions, each checked against the oracle."""
    s = configs.spec(1)
    b = configs.build(s)
    prob = O.Problem(**configs.oracle_problem(s, b))
    gop = b["gop"]
    rng = np.random.default_rng(77)
    outs = []
    ogop = prob.global_operator()
    shape = gop.window.shape
    for lo, hi in [((0, 0), (shape[0] - 1, shape[1] - 1)), ((1, 3), (shape[0] - 2, shape[1] - 1)),
                   ((5, 31), (22, 160))]:  # inclusive corners
        reg = Window(tuple(a + b for a, b in zip(gop.window.lo, lo)), tuple(a + b for a, b in zip(gop.window.lo, hi)))
        v = rng.standard_normal((5,) + reg.shape) + 1j * rng.standard_normal((5,) + reg.shape)
        got = gop.apply(v, region=reg)
        outs.append(np.asarray(got).ravel())
        for r in range(5):
            assert rel(got[r], ogop.apply(v[r], reg.lo)) <= 1e-14
    return np.concatenate(outs)


def test_stencil_apply_raster_kappa(cuda, raster):
    s, b, prob, oops = raster
    rng = np.random.default_rng(6)
    for idx in [(1, 1), (2, 2), (4, 1)]:
        op = b["ops"][idx]
        v = rng.standard_normal(op.window.shape) + 1j * rng.standard_normal(op.window.shape)
        assert rel(op.apply(v), oops[idx].apply(v)) <= 1e-14


@pytest.mark.parametrize("which,method", [("cfg1", "block-lu"), ("cfg1", "separable"),
                                          ("raster", "auto")])
def test_block_lu_solve_roundtrip(cuda, which, method, cfg1, raster):
    """Single-operator solves: block LU (K2/K3) and the modal backend
    (K2m/K3m, 'separable') vs the oracle's Schur/Sylvester or SuperLU solve."""
    s, b, prob, oops = cfg1 if which == "cfg1" else raster
    cache = FactorizationCache(method=method)
    rng = np.random.default_rng(7)
    for idx in list(b["ops"])[:4]:
        op = b["ops"][idx]
        fact = cache.get(op)
        assert fact.backend == ("splu" if method != "separable" else "separable")
        assert fact.device_backend == ("block-lu" if method != "separable" else "modal")
        rhs = rng.standard_normal((2,) + op.window.shape) + 1j * rng.standard_normal((2,) + op.window.shape)
        x = fact.solve(rhs)
        ref = O.factorize(oops[idx]).solve(rhs[0])
        assert rel(x[0], ref) <= TOL
        for r in range(2):
            res = float(np.linalg.norm(oops[idx].apply(x[r]) - rhs[r]) / np.linalg.norm(rhs[r]))
            assert res <= 1e-12, res


@pytest.mark.parametrize("method", ["auto", "block-lu"])
def test_ddm_cfg1_parity_and_events(cuda, cfg1, method):
    """'auto' runs the modal solve (separable operators), 'block-lu' K3."""
    s, b, prob, oops = cfg1
    f = configs.sources(s, b["grid"])
    u, rep = diagonal_sweep_solve(f[0], b["partition"], b["ops"], FactorizationCache(method=method),
                                  record_events=True, warn_collar=False)
    ref, orep = O.ddm_apply(prob, oops, O.Cache(), f[0], record=True)
    assert rel(u.values, ref) <= TOL
    assert rep.solves == orep["solves"] == 64
    assert rep.nonzero_solves == orep["nonzero_solves"]
    assert rep.discarded_sources == orep["discarded_sources"]
    assert rep.events == orep["events"]


def _compact_problem():
    # the reference's test_ddm fixture (pkg/tests/test_ddm.py:27-53)
    h = 0.01
    n = 141
    grid = make_grid(((0, h * (n - 1)),) * 2, (n, n))
    part = make_partition(grid, (3, 3), overlap_d_points=5, pml_width_points=10)
    kappa = 25.0
    profile = PmlProfile(10, 5, tuned_sigma_max(kappa, 10 * h))
    ops = build_operators(part, profile, constant_model(1.0), kappa)
    a, bb = part.breaks[0][1], part.breaks[0][2]
    c = grid.axis_coords(0)[(a + bb) // 2]
    f = gaussian_source(grid, (c, c), kappa)
    mask = np.zeros(grid.counts, dtype=bool)
    inner = tuple(slice(sl.start + 1, sl.stop - 1) for sl in part.owned_slices((2, 2)))
    mask[inner] = True
    f = np.where(mask, f, 0)
    prob = O.Problem(grid.extents, grid.counts, (3, 3), 5, 10, profile.sigma_max, 2, kappa,
                     ("const", 1.0))
    return grid, part, ops, f, prob


def test_ddm_emission_pattern_compact_source(cuda):
    """Golden emission pattern of pkg/tests/test_ddm.py:108-129 on the GPU."""
    grid, part, ops, f, prob = _compact_problem()
    u, report = diagonal_sweep_solve(f, part, ops, FactorizationCache(), record_events=True)
    emitted = {}
    for event in report.events:
        if event["nonzero"]:
            key = tuple(event["subdomain"])
            assert key not in emitted
            emitted[key] = (event["sweep"], event["sources_consumed"], event["sources_emitted"])
    assert emitted[(2, 2)] == (1, 0, 8)
    for edge in ((2, 3), (3, 2)):
        assert emitted[edge] == (1, 1, 2)
    assert emitted[(1, 2)] == (2, 1, 2)
    assert emitted[(2, 1)] == (3, 1, 2)
    for corner, sweep in (((3, 3), 1), ((1, 3), 2), ((3, 1), 3), ((1, 1), 4)):
        assert emitted[corner] == (sweep, 3, 0)
    oops = prob.operators()
    ref, _ = O.ddm_apply(prob, oops, O.Cache(), f)
    assert rel(u.values, ref) <= TOL


@pytest.fixture(scope="module")
def cfg2_oracle():
    """Config 2 (the headline): the oracle's u and counters for all 16 seeded
    RHS that bench.py times (~0.3 s per RHS on the box's host)."""
    s = configs.spec(2)
    b = configs.build(s)
    f = configs.sources(s, b["grid"])
    assert f.shape[0] == 16
    prob = O.Problem(**configs.oracle_problem(s, b))
    oops = prob.operators()
    cache = O.Cache()
    out = [O.ddm_apply(prob, oops, cache, f[r]) for r in range(f.shape[0])]
    return s, b, f, out


from parity_util import flush_subnormal_owned, subnormal_owned  # noqa: E402


def _check_batch(tag, u, reps, want, f=None, part=None, recheck=None, spec=2):
    """u within 1e-10 of the oracle for every RHS; counters exactly equal,
    except on RHS with subnormal-only owned source pieces, which must then
    match exactly once those pieces are flushed (`recheck(r, f_clean)` ->
    (nonzero, discarded) of the GPU path, compared with the oracle's)."""
    worst = 0.0
    rechecked = []
    for r, (ref, orep) in enumerate(want):
        e = rel(u[r], ref)
        worst = max(worst, e)
        assert e <= TOL, (tag, r, e)
        same = (reps[r].nonzero_solves == orep["nonzero_solves"]
                and reps[r].discarded_sources == orep["discarded_sources"])
        if same:
            continue
        assert f is not None and subnormal_owned(f[r], part), (tag, r, "counters differ")
        fc = flush_subnormal_owned(f[r], part)
        got = recheck(r, fc)
        cfg = configs.spec(spec)
        prob = O.Problem(**configs.oracle_problem(cfg, configs.build(cfg)))
        _, oc = O.ddm_apply(prob, prob.operators(), O.Cache(), fc)
        assert got == (oc["nonzero_solves"], oc["discarded_sources"]), (tag, r, got, oc["nonzero_solves"])
        rechecked.append(r)
    print(f"\n{tag}: {len(want)} RHS, worst relative L2 vs oracle {worst:.2e}; counters exact"
          + (f" (RHS {rechecked}: exact after flushing subnormal-only source pieces)" if rechecked else ""))


def test_ddm_cfg2_bench_paths_all_rhs(cuda, cfg2_oracle):
    """Exactly what bench.py times on config 2, all 16 RHS vs the oracle:
    `value` = the RHS-grouped device plan (`device_plan(..., grouped=True)`,
    `.apply` on RHS-outer device rows, default modal cache); `e2e` =
    `diagonal_sweep_solve` on a pinned host batch (ds_ddm_apply_host)."""
    import torch

    from paper_2002_05327_b200.ddm import SweepPlan, device_plan

    s, b, f, want = cfg2_oracle
    part, ops = b["partition"], b["ops"]
    cache = FactorizationCache()
    R = f.shape[0]
    dp_run = device_plan(part, ops, cache, SweepPlan.default(2), R, grouped=True)
    assert getattr(dp_run, "groups", 1) == 2
    fd = torch.from_numpy(f.reshape(R, -1)).cuda()

    def recheck(r, fc):
        _, rp = diagonal_sweep_solve(fc, part, ops, cache, warn_collar=False)
        return rp.nonzero_solves, rp.discarded_sources

    for _ in range(2):  # first call captures the graphs, the second replays them
        u, _ = dp_run.apply(fd)
        reps = _reports_of(dp_run, R, part)
        _check_batch("cfg2 device (grouped, graph)", u.cpu().numpy().reshape(f.shape), reps, want,
                     f, part, recheck)
    fp = torch.from_numpy(f).pin_memory()
    for _ in range(2):
        uh, reps = diagonal_sweep_solve(fp, part, ops, cache, warn_collar=False)
        assert not uh.values.is_cuda and uh.values.is_pinned()
        _check_batch("cfg2 pinned host (e2e)", uh.values.numpy(), reps, want, f, part, recheck)


def _reports_of(dp, R, part):
    from paper_2002_05327_b200.ddm import SweepPlan, _reports

    return _reports(dp, R, SweepPlan.default(part.dim), part, False, False)


def test_ddm_cfg2_block_lu_all_rhs(cuda, cfg2_oracle):
    """The block-LU backend (K2/K3) on the same 16 RHS."""
    s, b, f, want = cfg2_oracle
    cache = FactorizationCache(method="block-lu")
    u, reps = diagonal_sweep_solve(f, b["partition"], b["ops"], cache, warn_collar=False)

    def recheck(r, fc):
        _, rp = diagonal_sweep_solve(fc, b["partition"], b["ops"], cache, warn_collar=False)
        return rp.nonzero_solves, rp.discarded_sources

    _check_batch("cfg2 block-LU", u.values, reps, want, f, b["partition"], recheck)


def test_modal_guard_forced_fallback(cuda, cfg1):
    """modal_cond_max below every operator's cond(V): each separable operator
    falls back to the block LU (backend 'splu', reason recorded) and the DDM
    result is bitwise the block-LU backend's and within 1e-10 of the oracle."""
    s, b, prob, oops = cfg1
    f = configs.sources(s, b["grid"])[0]
    cache = FactorizationCache(modal_cond_max=1.0)
    u, rep = diagonal_sweep_solve(f, b["partition"], b["ops"], cache, warn_collar=False)
    assert cache.count == 16
    for fa in cache._store.values():
        assert fa.backend == "splu" and fa.device_backend == "block-lu"
        assert "cond(V)" in fa.fallback
    ub, _ = diagonal_sweep_solve(f, b["partition"], b["ops"], FactorizationCache(method="block-lu"),
                                 warn_collar=False)
    assert np.array_equal(u.values, ub.values)
    ref, orep = O.ddm_apply(prob, oops, O.Cache(), f)
    assert rel(u.values, ref) <= TOL
    assert rep.nonzero_solves == orep["nonzero_solves"]


def test_wide_window_guard_parity(cuda):
    """Wider windows than configs 1/2/4 (2x2 subdomains of a 321^2-node
    interior, windows ~193 nodes, sigma0 = 40): the eigenbases reach
    cond(V) ~ 1e5 and ||V^-1 V - I|| ~ 3e-9, so the guard sends those
    operators to the block LU; the DDM map stays within 1e-10 of the oracle.
    The unguarded modal path's error is printed for the record."""
    import math as _m

    s = configs.Spec("wide-2x2", ((0.0, 1.0),) * 2, (320, 320), 16, 16, (2, 2),
                     2 * _m.pi * 20, 2, "direct", "constant", 1,
                     centers=((0.3, 0.4), (0.62, 0.71)))
    b = configs.build(s)
    f = configs.sources(s, b["grid"])
    cache = FactorizationCache()
    u, reps = diagonal_sweep_solve(f, b["partition"], b["ops"], cache, warn_collar=False)
    fell = [fa.fallback for fa in cache._store.values() if fa.fallback]
    assert fell, "expected the guard to reject at least one eigenbasis"
    uu, _ = diagonal_sweep_solve(f, b["partition"], b["ops"], FactorizationCache(modal_cond_max=_m.inf),
                                 warn_collar=False)
    prob = O.Problem(**configs.oracle_problem(s, b))
    oops = prob.operators()
    oc = O.Cache()
    for r in range(f.shape[0]):
        ref, orep = O.ddm_apply(prob, oops, oc, f[r])
        e = rel(u.values[r], ref)
        print(f"\nwide windows rhs {r}: guarded {e:.2e} ({len(fell)} of {cache.count} operators on "
              f"the block LU), unguarded modal {rel(uu.values[r], ref):.2e}")
        assert e <= TOL, e
        assert reps[r].nonzero_solves == orep["nonzero_solves"]


def test_ddm_linearity_and_determinism(cuda, cfg1):
    s, b, prob, oops = cfg1
    rng = np.random.default_rng(1)
    shape = b["grid"].counts
    f1 = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    f2 = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    cache = FactorizationCache()
    batch = np.stack([2.5 * f1 + f2, f1, f2])
    u, _ = diagonal_sweep_solve(batch, b["partition"], b["ops"], cache, warn_collar=False)
    lhs = u.values[0]
    rhs = 2.5 * u.values[1] + u.values[2]
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(lhs) < 1e-10
    u2, _ = diagonal_sweep_solve(batch, b["partition"], b["ops"], cache, warn_collar=False)
    assert np.array_equal(u.values, u2.values)
    # dense random source: every subdomain solve is nonzero
    ref, _ = O.ddm_apply(prob, oops, O.Cache(), f1)
    assert rel(u.values[1], ref) <= TOL


def test_gmres_ddm_raster_parity(cuda, raster):
    s, b, prob, oops = raster
    f = configs.sources(s, b["grid"])
    part, ops, gop = b["partition"], b["ops"], b["gop"]
    cache = FactorizationCache()
    full = part.grid.full_window()

    def apply_m(v):
        return diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)[0].values

    x, reps = gmres_batched(lambda v: gop.apply(v, region=full), apply_m, f, tol=1e-6)
    ogop = prob.global_operator()
    ocache = O.Cache()
    for r in range(f.shape[0]):
        xr, orep = O.gmres_ddm(prob, oops, ogop, ocache, f[r])
        assert reps[r].n_iter == orep["n_iter"]
        assert reps[r].converged and orep["converged"]
        e = rel(x[r], xr)
        print(f"\nraster-mini GMRES rhs {r}: {reps[r].n_iter} iterations, x vs oracle {e:.2e}")
        assert e <= TOL, e
        np.testing.assert_allclose(reps[r].residuals, orep["residuals"], rtol=1e-6, atol=1e-12)


def test_gmres_unbatched_matches_batched(cuda, raster):
    s, b, prob, oops = raster
    f = configs.sources(s, b["grid"])[:1]
    part, ops, gop = b["partition"], b["ops"], b["gop"]
    cache = FactorizationCache()
    full = part.grid.full_window()

    def apply_m(v):
        return diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)[0].values

    x1, rep1 = gmres(lambda v: gop.apply(v, region=full), apply_m, f[0])
    xb, repb = gmres_batched(lambda v: gop.apply(v, region=full), apply_m, f)
    assert rep1.n_iter == repb[0].n_iter
    assert rel(x1, xb[0]) <= 1e-12


# ---------------------------------------------------------------- goldens
# direct comparisons with the reference's own outputs (tests/golden/)
from pathlib import Path
import json
GOLD = Path(__file__).resolve().parent / "golden"


def test_gpu_vs_reference_golden_cfg1(cuda, cfg1):
    s, b, prob, oops = cfg1
    g = np.load(GOLD / "ddm_cfg1.npz")
    f = configs.sources(s, b["grid"])[0]
    u, rep = diagonal_sweep_solve(f, b["partition"], b["ops"], FactorizationCache(),
                                  record_events=True, warn_collar=False)
    assert rel(u.values, g["u"]) <= TOL
    assert [rep.solves, rep.nonzero_solves, rep.discarded_sources] == list(g["counters"])
    assert rep.events == json.loads(str(g["events"]))


def test_gpu_vs_reference_golden_compact_and_random(cuda):
    grid, part, ops, f, prob = _compact_problem()
    g = np.load(GOLD / "ddm_compact.npz")
    assert np.array_equal(f, g["source"])
    rng = np.random.default_rng(2)
    fr = rng.normal(size=grid.counts) + 1j * rng.normal(size=grid.counts)
    u, reps = diagonal_sweep_solve(np.stack([f, fr]), part, ops, FactorizationCache(),
                                   record_events=True, warn_collar=False)
    assert rel(u.values[0], g["u"]) <= TOL
    assert rel(u.values[1], g["u_random"]) <= TOL
    assert reps[0].events == json.loads(str(g["events"]))


def test_octant_partials_converge_by_sweep(cuda):
    """collect_partials (the sweep-ordered plan): the running sum after each
    sweep is exact on that sweep's octant region up to the PML error
    (pkg/tests/test_ddm.py:144-155: subdomain counts [4, 2, 2, 1], relative
    error < 1e-3 against a global direct solve -- here the oracle's SuperLU
    of the global operator)."""
    from paper_2002_05327_b200.ddm import octant_exactness_check

    grid, part, ops, f, prob = _compact_problem()
    u_ref = O.SparseLU(prob.global_operator()).solve(f)
    u, report = diagonal_sweep_solve(f, part, ops, FactorizationCache(), collect_partials=True,
                                     warn_collar=False)
    assert len(report.partials) == 4
    checks = octant_exactness_check(report.partials, u_ref, part, (2, 2))
    assert [c["subdomains"] for c in checks] == [4, 2, 2, 1]
    for c in checks:
        assert c["relative_error"] < 1e-3
    # the last partial is the full sweep result; the pipelined plan (default,
    # different launch order) gives the same u up to summation order
    assert rel(np.asarray(report.partials[-1]), u.values) <= 1e-15
    u_pipe, _ = diagonal_sweep_solve(f, part, ops, FactorizationCache(), warn_collar=False)
    assert rel(u_pipe.values, u.values) <= 1e-12


def test_gpu_additive_vs_reference_golden(cuda):
    """additive_ddm_solve (ddm.py:294-349) on the same kernels: vs the
    reference's own outputs (tests/golden/make_golden_additive.py), counters,
    first_nonzero_step, and the reference's additive-vs-diagonal check
    (pkg/tests/test_ddm.py:132-141)."""
    from paper_2002_05327_b200 import additive_ddm_solve

    grid, part, ops, f, prob = _compact_problem()
    g = np.load(GOLD / "ddm_additive.npz")
    assert np.array_equal(f, g["source"])
    rng = np.random.default_rng(7)
    fr = rng.normal(size=grid.counts) + 1j * rng.normal(size=grid.counts)
    cache = FactorizationCache()
    u, reps = additive_ddm_solve(np.stack([f, fr]), part, ops, cache, warn_collar=False)
    assert rel(u.values[0], g["u"]) <= TOL
    assert rel(u.values[1], g["u_random"]) <= TOL
    assert [reps[0].solves, reps[0].nonzero_solves, reps[0].discarded_sources] == list(g["counters"])
    assert [reps[1].solves, reps[1].nonzero_solves, reps[1].discarded_sources] == \
        list(g["counters_random"])
    fns = {" ".join(map(str, k)): v for k, v in reps[0].first_nonzero_step.items()}
    assert fns == json.loads(str(g["first_nonzero_step"]))
    assert reps[0].first_nonzero_step[(2, 2)] == 1 and reps[0].first_nonzero_step[(1, 1)] == 3
    ud, _ = diagonal_sweep_solve(f, part, ops, cache, warn_collar=False)
    assert rel(u.values[0], ud.values) < 1e-12
    # single RHS in -> single report out, NumPy in -> NumPy out
    u1, rep1 = additive_ddm_solve(f, part, ops, cache, warn_collar=False)
    assert isinstance(u1.values, np.ndarray) and rep1.solves == reps[0].solves
    assert rel(u1.values, g["u"]) <= TOL


def test_gpu_vs_reference_golden_raster_gmres(cuda, raster):
    s, b, prob, oops = raster
    g = np.load(GOLD / "raster_mini.npz")
    f = configs.sources(s, b["grid"])[:1]
    part, ops, gop = b["partition"], b["ops"], b["gop"]
    cache = FactorizationCache()
    u, _ = diagonal_sweep_solve(f, part, ops, cache, warn_collar=False)
    assert rel(u.values[0], g["u_ddm"]) <= TOL
    full = part.grid.full_window()
    x, reps = gmres_batched(lambda v: gop.apply(v, region=full),
                            lambda v: diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)[0].values,
                            f)
    assert reps[0].n_iter == int(g["n_iter"])
    e = rel(x[0], g["x_gmres"])
    print(f"\nraster-mini GMRES vs reference golden: x {e:.2e}")
    assert e <= TOL, e


# ------------------------------------------------------------------- 3D
def mini3d():
    s = configs.Spec("mini-3d", ((0.0, 1.0),) * 3, (24, 24, 24), 4, 4, (2, 2, 2), 2 * np.pi * 3,
                     1, "direct", "constant", 9, centers=((0.3, 0.55, 0.4),))
    return s, configs.build(s)


@pytest.mark.parametrize("method", ["block-lu", "separable"])
def test_3d_blocked_factor_solve_roundtrip(cuda, method):
    """Blocked (panel + GEMM) factorization and staged solve, m = 625; the
    modal backend (two in-slab transforms per direction) on the same ops."""
    s, b = mini3d()
    prob = O.Problem(**configs.oracle_problem(s, b))
    cache = FactorizationCache(method=method)
    rng = np.random.default_rng(11)
    for idx in [(1, 1, 1), (2, 1, 2)]:
        op = b["ops"][idx]
        fact = cache.get(op)
        assert fact.block_size > 160
        rhs = rng.standard_normal((2,) + op.window.shape) + 1j * rng.standard_normal((2,) + op.window.shape)
        x = fact.solve(rhs)
        oop = prob.operator(prob.window(idx), prob.box(idx), prob.interior_box())
        for r in range(2):
            res = float(np.linalg.norm(oop.apply(x[r]) - rhs[r]) / np.linalg.norm(rhs[r]))
            assert res <= 1e-11, res
        assert rel(x[0], O.factorize(oop).solve(rhs[0])) <= TOL


@pytest.mark.parametrize("method", ["auto", "block-lu"])
def test_3d_ddm_vs_reference_golden_both_plans(cuda, method):
    from paper_2002_05327_b200 import SweepPlan

    s, b = mini3d()
    g = np.load(GOLD / "ddm_3d_mini.npz")
    f = configs.sources(s, b["grid"])[0]
    cache = FactorizationCache(method=method)
    u, rep = diagonal_sweep_solve(f, b["partition"], b["ops"], cache, record_events=True,
                                  warn_collar=False)
    assert rel(u.values, g["u"]) <= TOL
    assert [rep.solves, rep.nonzero_solves, rep.discarded_sources] == list(g["counters"])
    assert rep.events == json.loads(str(g["events"]))
    u2, _ = diagonal_sweep_solve(f, b["partition"], b["ops"], cache, plan=SweepPlan.alternate_3d(),
                                 warn_collar=False)
    assert rel(u2.values, g["u_alt"]) <= TOL


def test_cfg4_full_size_parity(cuda):
    """Config 4 at full size (109^3, 4x4x4, 8 RHS) on the path bench.py times:
    the default cache (modal factorization of all 64 windows, no sharing).
    RHS 0 and 1 against the oracle's separable (Schur/Sylvester) 3D solver,
    counters equal; all 8 RHS through linearity of the batched map (u of a
    combination of the 8 sources = the combination of their u) and bitwise
    determinism of a second application."""
    import time

    s = configs.spec(4)
    b = configs.build(s)
    f = configs.sources(s, b["grid"])
    R = f.shape[0]
    cache = FactorizationCache()
    t0 = time.time()
    cache.prepare([b["ops"][i] for i in b["partition"].subdomains()])
    tf = time.time() - t0
    assert cache.count == 64
    assert all(fa.backend == "separable" for fa in cache._store.values())
    t0 = time.time()
    u, reps = diagonal_sweep_solve(f, b["partition"], b["ops"], cache, warn_collar=False)
    ta = time.time() - t0
    u2, _ = diagonal_sweep_solve(f, b["partition"], b["ops"], cache, warn_collar=False)
    assert np.array_equal(u.values, u2.values)
    coef = np.random.default_rng(4).standard_normal(R) + 1j * np.random.default_rng(5).standard_normal(R)
    comb = np.tensordot(coef, f, axes=1)
    uc, _ = diagonal_sweep_solve(comb, b["partition"], b["ops"], cache, warn_collar=False)
    lin_err = rel(uc.values, np.tensordot(coef, u.values, axes=1))
    assert lin_err <= TOL, lin_err
    prob = O.Problem(**configs.oracle_problem(s, b))
    oops = prob.operators()
    ocache = O.Cache()
    want = [O.ddm_apply(prob, oops, ocache, f[r]) for r in (0, 1)]

    def recheck(r, fc):
        _, rp = diagonal_sweep_solve(fc, b["partition"], b["ops"], cache, warn_collar=False)
        return rp.nonzero_solves, rp.discarded_sources

    _check_batch("cfg4 (modal, unshared)", u.values[:2], reps[:2], want, f[:2], b["partition"],
                 recheck, spec=4)
    print(f"cfg4: factor {tf:.1f} s, one 8-RHS application {ta:.2f} s, "
          f"linearity (8 RHS) {lin_err:.2e}")


def test_cfg5r_gmres_vs_reference_golden(cuda):
    """Config 5r (3D raster, 57^2x45, 4x4x4, the oracle-feasible stand-in for
    config 5): batched GMRES-DDM vs the reference's own solution
    (tests/golden/make_golden_5r.py, 64 SuperLU factorizations, ~5 min CPU)."""
    import hashlib

    g = np.load(GOLD / "gmres_cfg5r.npz")
    s = configs.spec("5r")
    b = configs.build(s)
    f = configs.sources(s, b["grid"])
    assert hashlib.sha256(np.ascontiguousarray(f[0]).tobytes()).hexdigest() == str(g["source_sha"])
    part, ops, gop = b["partition"], b["ops"], b["gop"]
    cache = FactorizationCache()
    full = part.grid.full_window()
    x, reps = gmres_batched(lambda v: gop.apply(v, region=full),
                            lambda v: diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)[0].values,
                            f, tol=1e-6)
    assert reps[0].n_iter == int(g["n_iter"]) and reps[0].converged
    e = rel(x[0], g["x"])
    print(f"\ncfg5r GMRES vs reference golden: {reps[0].n_iter} iterations, x {e:.2e}")
    assert e <= TOL, e
    np.testing.assert_allclose(reps[0].residuals, g["residuals"], rtol=1e-6, atol=1e-12)
    assert all(r.converged for r in reps)


def test_cfg3_full_size_gmres_parity(cuda):
    """Config 3 at full size (1241x441, 16x8 raster windows) on the path
    bench.py times (batched GMRES over the RHS-grouped DDM preconditioner):
    RHS 0-3 against the oracle's SuperLU-based GMRES-DDM (iterations equal,
    solution <= 1e-10, residual history to 1e-6)."""
    s = configs.spec(3)
    b = configs.build(s)
    f = configs.sources(s, b["grid"])[:4]
    part, ops, gop = b["partition"], b["ops"], b["gop"]
    cache = FactorizationCache()
    full = part.grid.full_window()
    x, reps = gmres_batched(lambda v: gop.apply(v, region=full),
                            lambda v: diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)[0].values,
                            f, tol=1e-6)
    prob = O.Problem(**configs.oracle_problem(s, b))
    oops, ogop, ocache = prob.operators(), prob.global_operator(), O.Cache()
    for r in range(f.shape[0]):
        xr, orep = O.gmres_ddm(prob, oops, ogop, ocache, f[r])
        e = rel(x[r], xr)
        print(f"\ncfg3 rhs {r}: {reps[r].n_iter} iterations (oracle {orep['n_iter']}), x vs oracle {e:.2e}")
        assert reps[r].n_iter == orep["n_iter"] and reps[r].converged
        assert e <= TOL, e
        np.testing.assert_allclose(reps[r].residuals, orep["residuals"], rtol=1e-6, atol=1e-12)


def test_edge_cases_zero_sources_and_errors(cuda, cfg1):
    """Exactly-zero sources (every visit skipped, zero counters), GMRES with
    a zero right-hand side (krylov.py:58-64), and the reference's error
    behaviour for mismatched shapes / unknown methods."""
    from paper_2002_05327_b200 import ConfigurationError, factorize

    s, b, prob, oops = cfg1
    counts = b["grid"].counts
    z = np.zeros((2,) + counts, dtype=np.complex128)
    f = configs.sources(s, b["grid"])
    batch = np.concatenate([z[:1], f[:1], z[1:]])
    cache = FactorizationCache()
    u, reps = diagonal_sweep_solve(batch, b["partition"], b["ops"], cache, warn_collar=False)
    assert not np.any(u.values[0]) and not np.any(u.values[2])
    assert reps[0].nonzero_solves == 0 and reps[0].discarded_sources == 0
    assert reps[1].nonzero_solves > 0
    ref, _ = O.ddm_apply(prob, oops, O.Cache(), f[0])
    assert rel(u.values[1], ref) <= TOL
    gop, full = b["gop"], b["partition"].grid.full_window()
    x, rep = gmres(lambda v: gop.apply(v, region=full),
                   lambda v: diagonal_sweep_solve(v, b["partition"], b["ops"], cache,
                                                  warn_collar=False)[0].values, z[0])
    assert rep.converged and rep.residuals == [0.0] and rep.n_iter == 0 and not np.any(x)
    with pytest.raises(ConfigurationError):
        diagonal_sweep_solve(np.zeros((5, 5), complex), b["partition"], b["ops"], cache)
    op = b["ops"][(1, 1)]
    with pytest.raises(ConfigurationError):
        op.apply(np.zeros((3, 3), complex))
    with pytest.raises(ConfigurationError):
        cache.get(op).solve(np.zeros((4, 4), complex))
    with pytest.raises(ConfigurationError):
        factorize(op, "nope")


def test_many_rhs_chunking(cuda, cfg1):
    """More right-hand sides than one native launch takes (chunks of 256)."""
    s, b, prob, oops = cfg1
    rng = np.random.default_rng(3)
    counts = b["grid"].counts
    base = rng.standard_normal((3,) + counts) + 1j * rng.standard_normal((3,) + counts)
    coef = rng.standard_normal((260, 3))
    batch = np.einsum("rk,k...->r...", coef, base)
    u, reps = diagonal_sweep_solve(batch, b["partition"], b["ops"], FactorizationCache(),
                                   warn_collar=False)
    assert len(reps) == 260
    ub, _ = diagonal_sweep_solve(base, b["partition"], b["ops"], FactorizationCache(),
                                 warn_collar=False)
    want = np.einsum("rk,k...->r...", coef, ub.values)
    assert np.linalg.norm(u.values - want) / np.linalg.norm(want) < 1e-10


@pytest.mark.parametrize("nrhs", [1, 5, 17, 33])
def test_ragged_rhs_counts(cuda, cfg1, nrhs):
    """RHS counts that leave partial DMMA tiles and ragged RHS chunks (K3
    chunks of 16, step kernels with 1- and 4-column lanes): every RHS equals
    the same combination of three solved bases (the map is linear)."""
    s, b, prob, oops = cfg1
    rng = np.random.default_rng(40 + nrhs)
    counts = b["grid"].counts
    base = rng.standard_normal((3,) + counts) + 1j * rng.standard_normal((3,) + counts)
    coef = rng.standard_normal((nrhs, 3)) + 1j * rng.standard_normal((nrhs, 3))
    batch = np.einsum("rk,k...->r...", coef, base)
    cache = FactorizationCache()
    u, reps = diagonal_sweep_solve(batch, b["partition"], b["ops"], cache, warn_collar=False)
    ub, _ = diagonal_sweep_solve(base, b["partition"], b["ops"], cache, warn_collar=False)
    want = np.einsum("rk,k...->r...", coef, ub.values)
    assert len(reps) == nrhs
    assert np.linalg.norm(u.values - want) / np.linalg.norm(want) < 1e-10


def test_pinned_host_path_matches_device_path(cuda, cfg1):
    """ds_ddm_apply_host (chunked uploads / downloads overlapped with the
    sweep, graph replay keyed on the host buffers) is bitwise the device
    path, also on replay and with a second pair of host buffers."""
    import torch

    s, b, prob, oops = cfg1
    rng = np.random.default_rng(5)
    shape = (3,) + b["grid"].counts
    f = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    cache = FactorizationCache()
    u_dev, rep_dev = diagonal_sweep_solve(torch.from_numpy(f).cuda(), b["partition"], b["ops"], cache,
                                          warn_collar=False)
    ref = u_dev.values.cpu().numpy()
    for _ in range(2):
        for fp in (torch.from_numpy(f).pin_memory(), torch.from_numpy(f.copy()).pin_memory()):
            u_h, rep_h = diagonal_sweep_solve(fp, b["partition"], b["ops"], cache, warn_collar=False)
            assert not u_h.values.is_cuda
            assert np.array_equal(u_h.values.numpy(), ref)
            assert [r.nonzero_solves for r in rep_h] == [r.nonzero_solves for r in rep_dev]
    oref, _ = O.ddm_apply(prob, oops, O.Cache(), f[0])
    assert rel(ref[0], oref) <= TOL


def test_rhs_groups_bitwise_equal_to_one_plan(cuda, cfg1):
    """GroupedPlan (RHS groups on separate streams, the device path for
    batches >= 16 RHS) is bitwise the single-plan map, counters included."""
    import torch

    from paper_2002_05327_b200.ddm import SweepPlan, device_plan

    s, b, prob, oops = cfg1
    rng = np.random.default_rng(21)
    shape = (16,) + b["grid"].counts
    f = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    f[3] = 0.0  # an all-zero RHS inside a group
    fd = torch.from_numpy(f.reshape(16, -1)).cuda()
    cache = FactorizationCache()
    dg = device_plan(b["partition"], b["ops"], cache, SweepPlan.default(2), 16, grouped=True)
    d1 = device_plan(b["partition"], b["ops"], cache, SweepPlan.default(2), 16)
    assert getattr(dg, "groups", 1) >= 2 and getattr(d1, "groups", 1) == 1  # 2 by default, DS_RHS_GROUPS overrides
    ug, _ = dg.apply(fd)
    u1, _ = d1.apply(fd)
    assert torch.equal(ug, u1)
    cg, c1 = dg.counters(16), d1.counters(16)
    for k in c1:
        assert np.array_equal(cg[k], c1[k]), k
    oref, _ = O.ddm_apply(prob, oops, O.Cache(), f[0])
    assert rel(u1[0].cpu().numpy().reshape(b["grid"].counts), oref) <= TOL


def test_grouped_pinned_host_path(cuda, cfg1):
    """16 pinned host RHS: two RHS groups sweep concurrently with one shared
    upload / download pipeline (ds_ddm_apply_host_groups); bitwise the
    device path, counters included, also on graph replay."""
    import torch

    s, b, prob, oops = cfg1
    rng = np.random.default_rng(33)
    shape = (16,) + b["grid"].counts
    f = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    f[5] = 0.0
    cache = FactorizationCache()
    u_dev, rep_dev = diagonal_sweep_solve(torch.from_numpy(f).cuda(), b["partition"], b["ops"], cache,
                                          warn_collar=False)
    ref = u_dev.values.cpu().numpy()
    fp = torch.from_numpy(f).pin_memory()
    import os

    os.environ["DS_HOST_GROUPS"] = "1"
    try:
        runs = [diagonal_sweep_solve(fp, b["partition"], b["ops"], cache, warn_collar=False)
                for _ in range(3)]
    finally:
        del os.environ["DS_HOST_GROUPS"]
    for u_h, rep_h in runs:
        assert np.array_equal(u_h.values.numpy(), ref)
        assert [r.nonzero_solves for r in rep_h] == [r.nonzero_solves for r in rep_dev]
        assert [r.discarded_sources for r in rep_h] == [r.discarded_sources for r in rep_dev]


def test_transfer_kernel_variants_bitwise(cuda, cfg1):
    """The three source-transfer kernels (option "k4": 1 = one block per
    band, 2 = flattened records + tiles, 3 = RHS columns per thread, the 2D
    default) evaluate psi in the same order (v1 / v2 bitwise, v3 to FMA
    contraction); the assembly's RHS-column widths ("k6_rv" 1 / 2 / 4) are
    bitwise equal.  Fresh plans per variant (graphs keep the options they
    were recorded with)."""
    import torch

    from paper_2002_05327_b200 import _engine
    from paper_2002_05327_b200.ddm import SweepPlan

    s, b, prob, oops = cfg1
    rng = np.random.default_rng(8)
    f = rng.standard_normal((4,) + b["grid"].counts)
    fd = torch.from_numpy(f.astype(np.complex128).reshape(4, -1)).cuda()
    cache = FactorizationCache()

    def run(name, value):
        old = _engine.set_option(name, value)
        try:
            dp = _engine.DevicePlan(b["partition"], b["ops"], cache, SweepPlan.default(2).directions, 4,
                                    pipelined=True)
            u, _ = dp.apply(fd)
            return u.cpu().numpy()
        finally:
            _engine.set_option(name, old)

    outs = [run("k4", v) for v in (1, 2, 3)]
    # same evaluation order; v3's different code shape lets nvcc contract
    # the complex multiply-adds into FMAs differently -> equal to rounding
    assert np.array_equal(outs[0], outs[1])
    assert rel(outs[2], outs[1]) <= 1e-13
    k6 = [run("k6_rv", v) for v in (1, 2, 4)]
    assert np.array_equal(k6[0], k6[1]) and np.array_equal(k6[1], k6[2])


def test_context_options_validate(cuda):
    from paper_2002_05327_b200 import _engine
    from paper_2002_05327_b200.errors import ConfigurationError

    assert _engine.get_option("k1") == 4 and _engine.get_option("pdl") in (0, 1)
    with pytest.raises(ConfigurationError):
        _engine.set_option("k1", 3)
    with pytest.raises(ConfigurationError):
        _engine.set_option("no_such_option", 1)


def test_gmres_restart_longer_than_combine_limit(cuda, raster):
    """restart = 70 > 64 vectors per ds_vec_combine call: the basis update
    runs in chunks.  (1) The chunked combination of 70 random vectors equals
    the dense sum to 1e-14.  (2) DDM-preconditioned GMRES with an
    unreachable tolerance runs the full 70-step cycle (past convergence to
    rounding level) and x matches the oracle's GMRES to 1e-10."""
    import torch

    from paper_2002_05327_b200.krylov import _Vec

    rng = np.random.default_rng(70)
    n, R, K = 5000, 3, 70
    xs_h = rng.standard_normal((K, R, n)) + 1j * rng.standard_normal((K, R, n))
    c_h = rng.standard_normal((K, R)) + 1j * rng.standard_normal((K, R))
    y0 = rng.standard_normal((R, n)) + 1j * rng.standard_normal((R, n))
    xs = [torch.from_numpy(x).cuda() for x in xs_h]
    y = torch.from_numpy(y0).cuda()
    _Vec(n).combine(xs, torch.from_numpy(c_h).cuda(), y)
    want = y0 + np.einsum("kr,krn->rn", c_h, xs_h)
    assert np.linalg.norm(y.cpu().numpy() - want) <= 1e-14 * np.linalg.norm(want)

    s, b, prob, oops = raster
    f = configs.sources(s, b["grid"])[:1]
    part, ops, gop = b["partition"], b["ops"], b["gop"]
    cache = FactorizationCache()
    full = part.grid.full_window()
    x, reps = gmres_batched(lambda v: gop.apply(v, region=full),
                            lambda v: diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)[0].values,
                            f, tol=1e-300, restart=70, max_iter=70)
    assert reps[0].n_iter == 70 and not reps[0].converged
    ogop, ocache = prob.global_operator(), O.Cache()
    xr, orep = O.gmres(lambda v: ogop.apply(v), lambda v: O.ddm_apply(prob, oops, ocache, v)[0],
                       f[0], tol=1e-300, restart=70, max_iter=70)
    assert orep["n_iter"] == 70
    e = rel(x[0], xr)
    print(f"\nrestart 70 (DDM-preconditioned, 70 steps): x vs oracle {e:.2e}")
    assert e <= TOL, e


def test_pinned_strided_and_empty_batches(cuda, cfg1):
    """A strided view of a pinned batch goes through one packed pinned copy
    (not a pageable reshape) and equals the device path; an empty batch
    returns an empty field (an empty RHS shard of a multi-rank run)."""
    import torch

    s, b, prob, oops = cfg1
    rng = np.random.default_rng(12)
    shape = (4,) + b["grid"].counts
    f = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    cache = FactorizationCache()
    fp = torch.from_numpy(f).pin_memory()
    view = fp[::2]
    assert not view.is_contiguous()
    u_h, reps = diagonal_sweep_solve(view, b["partition"], b["ops"], cache, warn_collar=False)
    u_d, _ = diagonal_sweep_solve(torch.from_numpy(f[::2].copy()).cuda(), b["partition"], b["ops"],
                                  cache, warn_collar=False)
    assert np.array_equal(u_h.values.numpy(), u_d.values.cpu().numpy())
    assert len(reps) == 2
    u0, r0 = diagonal_sweep_solve(np.zeros((0,) + b["grid"].counts, np.complex128), b["partition"],
                                  b["ops"], cache, warn_collar=False)
    assert u0.values.shape == (0,) + b["grid"].counts and r0 == []
    t0, _ = diagonal_sweep_solve(torch.zeros((0,) + b["grid"].counts, dtype=torch.complex128,
                                             device="cuda"), b["partition"], b["ops"], cache,
                                 warn_collar=False)
    assert t0.values.is_cuda and t0.values.shape[0] == 0


@pytest.mark.parametrize("cfg", ["5r", "mini3d"])
def test_stencil_3d_ragged_regions(cuda, cfg):
    """3D K1 on the global operator over ragged regions (partial blocks at
    every face), 3 RHS: <= 1e-14 vs the oracle for raster (5r) and constant
    kappa^2."""
    if cfg == "5r":
        s = configs.spec("5r")
    else:
        s = configs.Spec("mini-3d", ((0.0, 1.0),) * 3, (20, 22, 18), 3, 3, (2, 2, 2),
                         2 * np.pi * 2, 1, "direct", "constant", 9, centers=((0.3, 0.55, 0.4),))
    b = configs.build(s)
    prob = O.Problem(**configs.oracle_problem(s, b))
    gop, ogop = b["gop"], prob.global_operator()
    shape = gop.window.shape
    rng = np.random.default_rng(33)
    for lo, hi in [((0, 0, 0), tuple(n - 1 for n in shape)),
                   ((1, 2, 3), (shape[0] - 2, shape[1] - 1, shape[2] - 3)),
                   ((3, 1, 0), (9, 6, 33 if shape[2] > 33 else shape[2] - 1))]:
        reg = Window(tuple(a + c for a, c in zip(gop.window.lo, lo)),
                     tuple(a + c for a, c in zip(gop.window.lo, hi)))
        v = rng.standard_normal((3,) + reg.shape) + 1j * rng.standard_normal((3,) + reg.shape)
        got = np.asarray(gop.apply(v, region=reg))
        for r in range(3):
            assert rel(got[r], ogop.apply(v[r], reg.lo)) <= 1e-14, (lo, hi, r)


@pytest.mark.parametrize("which", ["cfg1", "mini3d"])
@pytest.mark.parametrize("option", ["kskip"])
def test_transform_work_skips_exact(cuda, cfg1, which, option):
    """Option "kskip" (default on): the first forward transform of a modal
    visit walks only the 8-wide K-chunks that K6 marked nonzero; the
    skipped terms are products with exact zeros, so u equals the dense walk
    value for value (2D: config 1 with random and point sources; 3D: the
    2x2x2 mini problem, whose first pass runs along in-slab axis 1).  Fresh
    plans per setting (graphs keep the options they were recorded with)."""
    import torch

    from paper_2002_05327_b200 import _engine
    from paper_2002_05327_b200.ddm import SweepPlan

    if which == "cfg1":
        s, b = cfg1[0], cfg1[1]
        rng = np.random.default_rng(11)
        f = np.concatenate([rng.standard_normal((2,) + b["grid"].counts),
                            configs.sources(s, b["grid"], centers=[(0.3, 0.4), (0.8, 0.15)])])
        dim = 2
    else:
        s, b = mini3d()
        f = np.concatenate([configs.sources(s, b["grid"]),
                            np.random.default_rng(12).standard_normal((1,) + b["grid"].counts)])
        dim = 3
    R = f.shape[0]
    fd = torch.from_numpy(f.astype(np.complex128).reshape(R, -1)).cuda()
    cache = FactorizationCache()

    work = {}

    def run(value):
        old = _engine.set_option(option, value)
        try:
            dp = _engine.DevicePlan(b["partition"], b["ops"], cache, SweepPlan.default(dim).directions, R,
                                    pipelined=True)
            dp.enable_graph(False)  # a captured graph keeps the counter argument it was recorded with
            u, _ = dp.apply(fd)
            # the executed-work counter (ds_ctx_work, bench.py's roofline numerator)
            _engine.set_option("count_work", 1)
            _engine.executed_work(reset=True)
            u2, _ = dp.apply(fd)
            work[value] = (_engine.executed_work(reset=True), dp)
            _engine.set_option("count_work", 0)
            assert torch.equal(u, u2)
            return u.cpu().numpy()
        finally:
            _engine.set_option("count_work", 0)
            _engine.set_option(option, old)

    dense, sparse = run(0), run(1)
    assert np.array_equal(dense, sparse)
    assert np.count_nonzero(sparse) > 0
    # dense walk: n_b m (sum of in-slab extents) multiply-adds per transform
    # direction for every nonzero (visit, RHS) column; the sparse walk drops
    # the all-zero K-chunks of the first forward pass only
    cm_dense, dp = work[0]
    vnz = dp.counters(R)["visit_nonzero"]
    expect = 0
    for si, fct in enumerate(dp._keep[1]):
        per = 2 * fct.n_blocks * fct.block_size * (sum(fct.shape) - fct.shape[fct.block_axis])
        expect += per * int(vnz[:, si, :].sum())
    assert cm_dense == expect
    assert 0 < work[1][0] < cm_dense
    _engine.executed_work(reset=True)
    assert _engine.executed_work() == 0


def test_additive_cfg2_many_visits_per_launch(cuda):
    """The additive schedule visits every subdomain in every step: 64 modal
    visits per launch on config 2's 8 x 8 partition, i.e. more than the 32
    visits one transform / recurrence kernel launch tabulates (MG_MAXJ), so
    the launcher splits the list.  Two RHS (a seeded Gaussian and a random
    field) vs the oracle's additive restatement (ddm.py:294-349)."""
    from paper_2002_05327_b200 import additive_ddm_solve

    s = configs.spec(2)
    b = configs.build(s)
    grid, part, ops = b["grid"], b["partition"], b["ops"]
    rng = np.random.default_rng(21)
    f = np.stack([configs.sources(s, grid)[3],
                  rng.normal(size=grid.counts) + 1j * rng.normal(size=grid.counts)])
    u, reps = additive_ddm_solve(f, part, ops, FactorizationCache(), warn_collar=False)
    prob = O.Problem(**configs.oracle_problem(s, b))
    oops, cache = prob.operators(), O.Cache()
    for r in range(2):
        ref, orep = O.additive_apply(prob, oops, cache, f[r])
        e = rel(u.values[r], ref)
        assert e <= TOL, (r, e)
        assert reps[r].nonzero_solves == orep["nonzero_solves"], r
