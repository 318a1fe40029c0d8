#!/usr/bin/env python
"""Generate the golden fixtures of tests/golden/ by running the REFERENCE.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are the pinned synthetic inputs of SURVEY §8(d) (seeded NumPy,
recreated by paper_2002_05327_b200.configs); every fixture stores a
checksum of its input so the tests can prove they regenerate the same
bytes.  Outputs come from the reference's public API only
(`diagsweep.make_grid / make_partition / build_operators /
diagonal_sweep_solve / gmres`, `transfer.rule_allows / next_usable_sweep`).
Nothing here is copied from the reference sources.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import diagsweep as R  # noqa: E402  (the reference)
from diagsweep.ddm import SweepPlan as RPlan  # noqa: E402
from diagsweep.ddm import build_global_operator as r_bgo  # noqa: E402
from diagsweep.ddm import build_operators as r_bo  # noqa: E402
from diagsweep.media import RasterModel as RRaster  # noqa: E402
from diagsweep.transfer import next_usable_sweep as r_nus  # noqa: E402
from diagsweep.transfer import psi as r_psi  # noqa: E402
from diagsweep.transfer import rule_allows as r_rule  # noqa: E402

from paper_2002_05327_b200 import configs  # noqa: E402


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def ref_problem(spec_obj):
    b = configs.build(spec_obj)  # only for grid extents/counts, omega and raw c
    g = b["grid"]
    rg = R.make_grid(g.extents, g.counts)
    rp = R.make_partition(rg, spec_obj.counts, spec_obj.d, spec_obj.pml)
    prof = R.PmlProfile(spec_obj.pml, spec_obj.d, spec_obj.sigma_max, spec_obj.exponent)
    model = R.constant_model(1.0) if b["c"] is None else RRaster(tuple(spec_obj.interior), b["c"])
    ops = r_bo(rp, prof, model, b["omega"])
    gop = r_bgo(rp, prof, model, b["omega"])
    return b, rg, rp, ops, gop


def metadata(spec_obj, rp, ops):
    subs = list(rp.subdomains())
    dim = rp.dim
    dirs = [d for d in itertools.product((-1, 0, 1), repeat=dim) if any(d)]
    plan = RPlan.default(dim).directions
    meta = {
        "counts": list(rp.grid.counts), "extents": [list(e) for e in rp.grid.extents],
        "breaks": [list(b) for b in rp.breaks], "subdomains": [list(s) for s in subs],
        "window": [], "box": [], "owned": [], "support": [], "beta_sha": [],
        "alpha_sha": [], "kappa2_sha": [], "fingerprint": [],
        "steps": {}, "routing": {}, "bands": {},
    }
    for idx in subs:
        w, b = rp.window(idx), rp.box(idx)
        meta["window"].append([list(w.lo), list(w.hi)])
        meta["box"].append([list(b.lo), list(b.hi)])
        meta["owned"].append([[s.start, s.stop] for s in rp.owned_slices(idx)])
        sw, sv = rp.beta00_support(idx)
        meta["support"].append([list(sw.lo), list(sw.hi)])
        meta["beta_sha"].append(sha(sv))
        op = ops[idx]
        meta["alpha_sha"].append(sha(np.concatenate([*op.alpha_nodes, *op.alpha_faces])))
        k2 = op.kappa2 if op.kappa2_kind != "axis" else op.kappa2[1]
        meta["kappa2_sha"].append(sha(np.asarray(k2, dtype=np.float64)))
        meta["fingerprint"].append(op.fingerprint)
    for sweep, sd in enumerate(plan, 1):
        groups = {}
        for idx in subs:
            groups.setdefault(R.partition.sweep_step_of(idx, sd, rp.counts), []).append(list(idx))
        meta["steps"][str(sweep)] = {str(k): sorted(v) for k, v in groups.items()}
        meta["routing"][str(sweep)] = {
            " ".join(map(str, d)): r_nus(d, sweep, plan) for d in dirs}
    # psi band windows for every in-range (source, direction): geometry of
    # the reference's own psi on a zero field
    for idx in subs:
        win = rp.window(idx)
        zero = np.zeros(win.shape, dtype=np.complex128)
        for d in dirs:
            ts = r_psi(rp, ops, idx, d, zero, zero)
            key = " ".join(map(str, idx)) + "|" + " ".join(map(str, d))
            meta["bands"][key] = None if ts is None else [list(ts.window.lo), list(ts.window.hi)]
    return meta


def ddm_case(rp, ops, f, record=True):
    cache = R.FactorizationCache()
    u, rep = R.diagonal_sweep_solve(f, rp, ops, cache, record_events=record, warn_collar=False)
    return u.values, rep


def main():
    out = {}
    # ---- rule tables (pins routing; also checked against pkg/tests/data/*.csv)
    tables = {}
    for dim in (2, 3):
        dirs = [d for d in itertools.product((-1, 0, 1), repeat=dim) if any(d)]
        sweeps = list(itertools.product((-1, 1), repeat=dim))
        rows = [(s, g, u, int(r_rule(s, g, u, dim))) for s in dirs for g in sweeps for u in sweeps]
        tables[f"rule_{dim}d"] = np.array([list(s) + list(g) + list(u) + [a] for s, g, u, a in rows],
                                          dtype=np.int8)
    np.savez_compressed(HERE / "rule_tables.npz", **tables)

    # ---- metadata of every config (bit-exact index maps, coefficient hashes)
    for k in (1, 2, 3, 4, 5, "5r"):
        s = configs.spec(k)
        b, rg, rp, ops, gop = ref_problem(s)
        meta = metadata(s, rp, ops)
        meta["omega"] = b["omega"]
        meta["gop_alpha_sha"] = sha(np.concatenate([*gop.alpha_nodes, *gop.alpha_faces]))
        f = configs.sources(s, b["grid"])
        meta["source_sha"] = sha(f)
        meta["velocity_sha"] = None if b["c"] is None else sha(b["c"])
        (HERE / f"meta_cfg{k}.json").write_text(json.dumps(meta, separators=(",", ":")))
        print("meta", k, len(meta["subdomains"]), "subdomains")

    # ---- DDM solutions
    s = configs.spec(1)
    b, rg, rp, ops, gop = ref_problem(s)
    f = configs.sources(s, b["grid"])
    u, rep = ddm_case(rp, ops, f[0])
    np.savez_compressed(HERE / "ddm_cfg1.npz", u=u, source_sha=sha(f[0]),
                        counters=np.array([rep.solves, rep.nonzero_solves, rep.discarded_sources]),
                        events=json.dumps(rep.events))
    print("ddm cfg1", rep.nonzero_solves)

    # reference test fixture geometry (pkg/tests/test_ddm.py:27-53), compact source
    h, n = 0.01, 141
    grid = R.make_grid(((0, h * (n - 1)),) * 2, (n, n))
    part = R.make_partition(grid, (3, 3), overlap_d_points=5, pml_width_points=10)
    kappa = 25.0
    prof = R.PmlProfile(10, 5, R.tuned_sigma_max(kappa, 10 * h))
    ops2 = r_bo(part, prof, R.constant_model(1.0), kappa)
    a, bb = part.breaks[0][1], part.breaks[0][2]
    c = grid.axis_coords(0)[(a + bb) // 2]
    src = R.gaussian_source(grid, (c, c), kappa)
    mask = np.zeros(grid.counts, dtype=bool)
    inner = tuple(slice(sl.start + 1, sl.stop - 1) for sl in part.owned_slices((2, 2)))
    mask[inner] = True
    src = np.where(mask, src, 0)
    u2, rep2 = ddm_case(part, ops2, src)
    rng = np.random.default_rng(2)
    frand = rng.normal(size=grid.counts) + 1j * rng.normal(size=grid.counts)
    u3, rep3 = ddm_case(part, ops2, frand, record=False)
    np.savez_compressed(HERE / "ddm_compact.npz", u=u2, source=src, sigma_max=prof.sigma_max,
                        counters=np.array([rep2.solves, rep2.nonzero_solves, rep2.discarded_sources]),
                        events=json.dumps(rep2.events), u_random=u3, random_sha=sha(frand))
    print("ddm compact", rep2.nonzero_solves)

    # heterogeneous (raster) mini problem: DDM + GMRES
    mini = configs.Spec("mini-raster", ((0.0, 2.4), (0.0, 0.8)), (240, 80), 10, 10, (4, 2),
                        None, 3, "gmres", "raster", 3, c_range=(1.5, 3.0), noise=0.15,
                        filt=10.0, src_depth_h=5.0)
    b, rg, rp, ops, gop = ref_problem(mini)
    f = configs.sources(mini, b["grid"])
    u4, rep4 = ddm_case(rp, ops, f[0], record=False)
    cache = R.FactorizationCache()
    full = rp.grid.full_window()
    x, srep = R.gmres(lambda v: gop.apply(v, region=full),
                      lambda v: R.diagonal_sweep_solve(v, rp, ops, cache, warn_collar=False)[0].values,
                      f[0], tol=1e-6, restart=30, max_iter=200)
    np.savez_compressed(HERE / "raster_mini.npz", u_ddm=u4, x_gmres=x,
                        residuals=np.array(srep.residuals), n_iter=srep.n_iter,
                        converged=srep.converged, source_sha=sha(f[0]), velocity_sha=sha(b["c"]))
    print("raster mini gmres iterations", srep.n_iter)

    # small 3D constant case (2x2x2, both sweep orders)
    s3 = configs.Spec("mini-3d", ((0.0, 1.0),) * 3, (24, 24, 24), 4, 4, (2, 2, 2), 2 * np.pi * 3,
                      1, "direct", "constant", 9, centers=((0.3, 0.55, 0.4),))
    b, rg, rp, ops, gop = ref_problem(s3)
    f = configs.sources(s3, b["grid"])
    u5, rep5 = ddm_case(rp, ops, f[0])
    cache = R.FactorizationCache()
    u6, _ = R.diagonal_sweep_solve(f[0], rp, ops, cache, plan=RPlan.alternate_3d(), warn_collar=False)
    np.savez_compressed(HERE / "ddm_3d_mini.npz", u=u5, u_alt=u6.values, source_sha=sha(f[0]),
                        counters=np.array([rep5.solves, rep5.nonzero_solves, rep5.discarded_sources]),
                        events=json.dumps(rep5.events))
    print("3d mini", rep5.nonzero_solves)


if __name__ == "__main__":
    main()
