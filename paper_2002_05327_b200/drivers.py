"""Drivers on the batched GPU DDM (reference cli.py).

The reference drives its sweep one right-hand side at a time from host
loops (`_solve_once` cli.py:63-104, `decay_history` cli.py:175-191,
`cmd_precond_study` cli.py:256-298).  Here every driver takes a source
batch `[R, *counts]` (or one field, as the reference) and keeps the loop on
the device: the residual r = f - A u (K1 stencil), its norms (K7) and the
DDM correction stay in HBM, and the host reads one residual table per call
instead of one norm per iteration.  Results, iteration counts and file
artifacts are those of the reference for a single RHS
(tests/test_drivers.py, tests/test_gpu_drivers.py against the reference's
own CLI output).
"""

from __future__ import annotations

import time

import numpy as np

from .ddm import build_global_operator, build_operators, diagonal_sweep_solve
from .errors import ConfigurationError, SolverError
from .grid import ComplexField
from .krylov import gmres, gmres_batched
from .media import point_shots
from .subdomain import FactorizationCache, factorize

MODES = ("direct-ddm", "gmres-ddm", "global-direct")


def build_problem(cfg, cells=None, partition_counts=None):
    """grid, partition, subdomain operators and global operator of a run
    (cli.py:51-60)."""
    grid = cfg.build_grid(cells)
    partition = cfg.build_partition(grid, partition_counts)
    profile = cfg.build_profile()
    model = cfg.build_model()
    ops = build_operators(partition, profile, model, cfg.omega)
    gop = build_global_operator(partition, profile, model, cfg.omega)
    return grid, partition, ops, gop


def _device(f, counts):
    """(batch [R, *counts] on cuda, batched?) without copying device input."""
    import torch

    if not torch.cuda.is_available():
        raise SolverError("no CUDA device: the B200 path has no CPU fallback")
    t = f if hasattr(f, "detach") else torch.from_numpy(np.ascontiguousarray(f, np.complex128))
    batched = tuple(t.shape[1:]) == tuple(counts)
    if not batched and tuple(t.shape) != tuple(counts):
        raise ConfigurationError("source shape does not match the grid")
    t = t.to("cuda", torch.complex128)
    return (t if batched else t.reshape((1,) + tuple(counts))), batched


def _rel_residuals(gop, full, u, f):
    """||A u - f|| / ||f|| per RHS, on the device (one K1 launch)."""
    import torch

    R = f.shape[0]
    r = gop.apply(u, region=full) - f
    return (torch.linalg.vector_norm(r.reshape(R, -1), dim=1)
            / torch.linalg.vector_norm(f.reshape(R, -1), dim=1))


def solve_once(cfg, f, partition, operators, gop, record_events=False, cache=None):
    """One configured solve (cli.py:63-104), batched over RHS.

    Returns (u ComplexField on the host, info dict, DDM report(s) or None,
    GMRES report(s) or None).  For a batch, the per-RHS entries of `info`
    ("n_iter", "converged", "final_residual", "residual") are lists."""
    import torch

    mode = cfg.get("solver", "mode")
    if mode not in MODES:
        raise ConfigurationError(f"unknown solver mode {mode!r}")
    cache = FactorizationCache() if cache is None else cache
    full = partition.grid.full_window()
    counts = partition.grid.counts
    fd, batched = _device(f, counts)
    info = {"mode": mode, "config_sha256": cfg.sha256}
    ddm_rep = kry = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "global-direct":
        u = factorize(gop).solve(fd)
    elif mode == "direct-ddm":
        uf, ddm_rep = diagonal_sweep_solve(fd, partition, operators, cache,
                                           record_events=record_events)
        u = uf.values
    else:
        def apply_m(v):
            return diagonal_sweep_solve(v, partition, operators, cache, warn_collar=False)[0].values

        u, kry = gmres_batched(lambda v: gop.apply(v, region=full), apply_m, fd,
                               tol=cfg.getfloat("solver", "tol"),
                               restart=cfg.getint("solver", "restart"),
                               max_iter=cfg.getint("solver", "max_iter"))
        info["n_iter"] = [k.n_iter for k in kry]
        info["converged"] = [k.converged for k in kry]
        info["final_residual"] = [k.residuals[-1] for k in kry]
    torch.cuda.synchronize()
    info["wall_time"] = time.perf_counter() - t0
    info["residual"] = [float(x) for x in _rel_residuals(gop, full, u, fd).cpu()]
    vals = u.cpu().numpy()
    if not batched:
        vals = vals[0]
        for k in ("n_iter", "converged", "final_residual", "residual"):
            if k in info:
                info[k] = info[k][0]
        ddm_rep = ddm_rep[0] if isinstance(ddm_rep, list) else ddm_rep
        kry = kry[0] if kry is not None else None
    return ComplexField(partition.grid, vals), info, ddm_rep, kry


def decay_history(cfg, counts, f=None, n_it=None, cache=None):
    """Iterative-mode residual decay for one partition (cli.py:175-191):
    u_0 = 0, r_k = f - A u_k, u_{k+1} = u_k + DDM(r_k); returns
    ||r_k|| / ||f|| for k < n_it -- `[n_it]` for one source, `[R, n_it]` for
    a batch.  The loop runs on the device; norms are read once at the end."""
    import torch

    grid, partition, ops, gop = build_problem(cfg, partition_counts=counts)
    if f is None:
        f = cfg.build_source(grid)
    n_it = n_it or cfg.getint("decay", "iterations")
    cache = FactorizationCache() if cache is None else cache
    full = grid.full_window()
    fd, batched = _device(f, grid.counts)
    R = fd.shape[0]
    nf = torch.linalg.vector_norm(fd.reshape(R, -1), dim=1)
    u = torch.zeros_like(fd)
    hist = torch.empty((n_it, R), dtype=torch.float64, device=fd.device)
    for k in range(n_it):
        r = fd - gop.apply(u, region=full)
        hist[k] = torch.linalg.vector_norm(r.reshape(R, -1), dim=1) / nf
        du, _ = diagonal_sweep_solve(r, partition, ops, cache, warn_collar=False)
        u += du.values
    h = hist.T.cpu().numpy()
    return h if batched else h[0]


def fit_decay_rate(history, skip: int, floor: float) -> float:
    """Least-squares slope of log10(residual) over the iterations above the
    stagnation floor, after skipping the first `skip` of them (cli.py:194-201)."""
    h = np.asarray(history, dtype=np.float64)
    keep = np.flatnonzero(h > floor)[skip:]
    if keep.size < 2:
        raise SolverError("too few iterations above the floor to fit a rate")
    return float(np.polyfit(keep, np.log10(h[keep]), 1)[0])


def precond_rows(cfg):
    """[precond] rows = "cells,NxM,frequency; ..." -> [(cells, counts, freq)]."""
    rows = []
    for tok in (t.strip() for t in cfg.get("precond", "rows").split(";")):
        if not tok:
            continue
        try:
            c, p, fr = (x.strip() for x in tok.split(","))
            rows.append((int(c), tuple(int(x) for x in p.split("x")), float(fr)))
        except ValueError:
            raise ConfigurationError(f"bad precond row {tok!r}") from None
    return rows


def precond_case(cfg, cells, counts, freq):
    """The sub-configuration and four-shot source of one study row
    (cli.py:272-287): gmres-ddm, shots at the (1/4, 3/4) lattice of the
    interior box."""
    sub = cfg.with_values(problem={"frequency": repr(freq)},
                          partition={"counts": ",".join(map(str, counts))},
                          discretization={"interior_cells": str(cells)},
                          solver={"mode": "gmres-ddm"})
    grid, partition, ops, gop = build_problem(sub, (cells,) * sub.dim)
    box = sub.interior_extents()
    shots = [tuple(a + t * (b - a) for (a, b), t in zip(box, frac))
             for frac in ((0.25, 0.25), (0.25, 0.75), (0.75, 0.25), (0.75, 0.75))]
    return sub, grid, partition, ops, gop, point_shots(grid, shots, box)


def precond_study(cfg):
    """GMRES-DDM iteration counts over the [precond] rows (cli.py:256-298):
    [(cells, "NxM", frequency, n_iter, converged, wall_time)]."""
    out = []
    for cells, counts, freq in precond_rows(cfg):
        sub, grid, partition, ops, gop, f = precond_case(cfg, cells, counts, freq)
        _, info, _, _ = solve_once(sub, f, partition, ops, gop)
        out.append((cells, "x".join(map(str, counts)), freq, info["n_iter"], info["converged"],
                    info["wall_time"]))
    return out


__all__ = ["MODES", "build_problem", "decay_history", "fit_decay_rate", "gmres",
           "precond_case", "precond_rows", "precond_study", "solve_once"]
