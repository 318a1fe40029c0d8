"""The diagonal sweeping DDM engine — drop-in for `diagsweep.ddm`.

`diagonal_sweep_solve(f, partition, operators, cache, plan=None, *,
collect_partials, record_events, record_transfers, warn_collar)` keeps the
reference signature (diagsweep/ddm.py:212-223) and additionally accepts a
leading right-hand-side batch axis: `f` of shape `[*grid.counts]` returns
`(ComplexField, DdmReport)` exactly like the reference; `f` of shape
`[R, *grid.counts]` returns `(ComplexField [R, *counts], [DdmReport] * R)`.
NumPy input gives NumPy output; a torch CUDA tensor stays on the device.

Everything between the input and the output runs in one native call
(`ds_ddm_apply`): per anti-diagonal step one RHS-assembly kernel, one
batched block-substitution launch for every subdomain on the step and every
RHS, one beta00 accumulation kernel and one fused transfer kernel.  The
emission masks of the reference (`content_cuts`/`solve_cuts`/`emits`,
ddm.py:82-110, and the exact-zero tests at ddm.py:248/256) are evaluated on
the device per RHS; the host-side functions below are the same rules on
frozensets, kept for API compatibility and for the report.
"""

from __future__ import annotations

import itertools
import json
import os
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError
from .grid import ComplexField, Window
from .partition import Partition, octant_region, steps_per_sweep, sweep_step_of
from .pml import PmlProfile, assemble_operator
from .subdomain import FactorizationCache
from .transfer import next_usable_sweep

_DEFAULT_2D = ((1, 1), (-1, 1), (1, -1), (-1, -1))
_DEFAULT_3D = (
    (1, 1, 1), (-1, 1, 1), (1, -1, 1), (-1, -1, 1),
    (1, 1, -1), (-1, 1, -1), (1, -1, -1), (-1, -1, -1),
)
_ALTERNATE_3D = (
    (1, 1, 1), (-1, 1, 1), (1, -1, 1), (1, 1, -1),
    (-1, -1, 1), (-1, 1, -1), (1, -1, -1), (-1, -1, -1),
)


@dataclass(frozen=True)
class SweepPlan:
    """Ordered diagonal sweep directions (ddm.py:48-72)."""

    directions: tuple

    def __post_init__(self):
        dim = len(self.directions[0])
        want = set(itertools.product((-1, 1), repeat=dim))
        if set(self.directions) != want or len(self.directions) != len(want):
            raise ConfigurationError("sweep plan must cover every diagonal direction exactly once")

    @classmethod
    def default(cls, dim: int) -> "SweepPlan":
        return cls(_DEFAULT_2D if dim == 2 else _DEFAULT_3D)

    @classmethod
    def alternate_3d(cls) -> "SweepPlan":
        return cls(_ALTERNATE_3D)

    @property
    def dim(self) -> int:
        return len(self.directions[0])


def source_directions(dim: int):
    """The 3^dim - 1 transfer directions in itertools.product order."""
    return tuple(d for d in itertools.product((-1, 0, 1), repeat=dim) if any(d))


def content_cuts(direction, parent_cuts: frozenset) -> frozenset:
    out = {(a, -c) for a, c in enumerate(direction) if c}
    out |= {(a, s) for (a, s) in parent_cuts if direction[a] == 0}
    return frozenset(out)


def solve_cuts(arrival_cuts, has_own_source: bool) -> frozenset:
    if has_own_source or not arrival_cuts:
        return frozenset()
    return frozenset.intersection(*arrival_cuts)


def emits(direction, cuts: frozenset) -> bool:
    return not any(c != 0 and (a, c) in cuts for a, c in enumerate(direction))


def cut_mask_to_set(mask: int, dim: int) -> frozenset:
    """Decode the device cut bitmask (bit 2a + (side > 0))."""
    return frozenset((a, 1 if s else -1) for a in range(dim) for s in (0, 1)
                     if mask >> (2 * a + s) & 1)


def build_operators(partition: Partition, profile: PmlProfile, velocity, omega: float,
                    assembly: str = "host") -> dict:
    clamp = partition.interior_box()
    return {
        index: assemble_operator(partition.grid, partition.window(index), partition.box(index),
                                 profile, velocity, omega, clamp_box=clamp, assembly=assembly)
        for index in partition.subdomains()
    }


def build_global_operator(partition: Partition, profile: PmlProfile, velocity, omega,
                          assembly: str = "host"):
    return assemble_operator(partition.grid, partition.grid.full_window(), partition.interior,
                             profile, velocity, omega, clamp_box=partition.interior_box(),
                             assembly=assembly)


@dataclass
class DdmReport:
    """Counters of one DDM application for one RHS (ddm.py:149-165)."""

    solves: int = 0
    nonzero_solves: int = 0
    discarded_sources: int = 0
    wall_time: float = 0.0
    events: list | None = None
    partials: list | None = None
    transfer_records: list | None = None
    first_nonzero_step: dict = field(default_factory=dict)

    def write_event_log(self, path) -> None:
        with open(path, "w") as fh:
            for event in self.events or []:
                fh.write(json.dumps(event) + "\n")


def restrict_source(f: np.ndarray, partition: Partition, warn_collar: bool = True) -> dict:
    """Owned pieces of a host source (ddm.py:168-195); the device engine uses
    the same owned windows (`Partition.owned_window`)."""
    if f.shape != partition.grid.counts:
        raise ConfigurationError("source shape does not match the grid")
    if warn_collar:
        _warn_collar(f, partition)
    out = {}
    for index in partition.subdomains():
        win = partition.owned_window(index)
        out[index] = (win, np.ascontiguousarray(f[win.slices()], dtype=np.complex128))
    return out


def _warn_collar(f, partition: Partition):
    inner = partition.interior.slices()
    if hasattr(f, "detach"):
        import torch

        probe = f.clone()
        probe[(Ellipsis,) + inner] = 0
        leak = bool(torch.any(probe != 0))
    else:
        probe = np.array(f, copy=True)
        probe[(Ellipsis,) + inner] = 0
        leak = bool(np.any(probe))
    if leak:
        warnings.warn("source support leaks into the global PML collar")


def _plan_key(partition, operators, directions, schedule="diagonal", pipelined=False):
    return (partition, tuple(id(operators[i]) for i in partition.subdomains()), directions,
            schedule, pipelined)


def _group_count(partition, nrhs: int, operators=None) -> int:
    """RHS groups for the device path: 2D batches of >= 16 RHS run as 2
    groups (measured: config 2 +8%, config 3 +15%; 3D batches gain nothing);
    raster (block-LU) batches of >= 64 RHS as 4 (config 3 with 9-CTA K3
    clusters: 155.4 vs 151.9 RHS/s; config 2's modal solve is best at 2).
    DS_RHS_GROUPS overrides."""
    env = os.environ.get("DS_RHS_GROUPS")
    if env:
        return max(1, int(env))
    if partition.dim != 2 or nrhs < 16:
        return 1
    raster = operators is not None and any(
        getattr(operators[i], "kappa2_kind", None) == "full" for i in partition.subdomains())
    return 4 if raster and nrhs >= 64 else 2


def device_plan(partition, operators, cache: FactorizationCache, plan: SweepPlan | None,
                nrhs: int, schedule: str = "diagonal", pipelined: bool | None = None,
                grouped: bool = False):
    """The cached native plan for (partition, operators, sweep order, schedule).

    pipelined (diagonal schedule; default on, DS_PIPELINE=0 turns it off):
    visits of different sweeps share a launch as soon as their sources are
    done (`_engine.launch_schedule`); the map is unchanged, sums stay
    deterministic.  Per-sweep partials need the sweep-ordered plan."""
    from . import _engine

    plan = plan or SweepPlan.default(partition.dim)
    directions = plan.directions if schedule == "diagonal" else ()
    if pipelined is None:
        pipelined = schedule == "diagonal" and os.environ.get("DS_PIPELINE", "1") != "0"
    pipelined = bool(pipelined) and schedule == "diagonal"
    G = _group_count(partition, nrhs, operators) if grouped and schedule == "diagonal" else 1
    key = _plan_key(partition, operators, directions, schedule, pipelined) + (("groups", G),)
    dp = cache._plans.get(key)
    if dp is None or dp.nrhs_max < nrhs:
        nmax = max(nrhs, dp.nrhs_max if dp else 0)
        slots = None
        if schedule == "diagonal":
            slots = cache.pool_slots([operators[i] for i in partition.subdomains()])
        if slots is not None:  # factors exceed HBM: pooled, launch-by-launch plan
            dp = None
            cache._plans.pop(key, None)
            dp = _engine.DevicePlan(partition, operators, cache, directions, nmax, schedule,
                                    pipelined=True, pool_slots=slots)
        elif G > 1:
            per = -(-nmax // G)
            dp = _engine.GroupedPlan([_engine.DevicePlan(partition, operators, cache, directions, per,
                                                         schedule, pipelined=pipelined)
                                      for _ in range(G)])
        else:
            dp = _engine.DevicePlan(partition, operators, cache, directions, nmax, schedule,
                                    pipelined=pipelined)
        cache._plans[key] = dp
    return dp


def diagonal_sweep_solve(f, partition: Partition, operators: dict,
                         cache: FactorizationCache | None = None, plan: SweepPlan | None = None,
                         *, collect_partials: bool = False, record_events: bool = False,
                         record_transfers: bool = False, warn_collar: bool = True):
    """One application of the diagonal sweeping DDM (batched over RHS)."""
    from . import _engine

    t0 = time.perf_counter()
    counts = partition.grid.counts
    shape = tuple(f.shape)
    if shape != counts and shape[1:] != counts:
        raise ConfigurationError("source shape does not match the grid")
    if cache is None:
        cache = FactorizationCache()
    if not isinstance(cache, FactorizationCache):
        raise ConfigurationError("cache must be a paper_2002_05327_b200 FactorizationCache")
    if warn_collar:
        _warn_collar(f, partition)
    plan = plan or SweepPlan.default(partition.dim)
    if (_engine.is_pinned_host(f) and not collect_partials
            and (f.shape[0] if shape[1:] == counts else 1) <= 256):
        # pinned host sources: uploads / downloads overlapped with the sweep
        # inside the library (ds_ddm_apply_host); result in pinned memory
        import torch

        batched = shape[1:] == counts
        fh = f
        if fh.dtype != torch.complex128 or not fh.is_contiguous():
            # a strided or non-complex128 view: one packed pinned copy (a
            # reshape would otherwise copy it silently into pageable memory)
            fh = fh.to(torch.complex128).contiguous().pin_memory()
        fh = fh.reshape(-1, int(np.prod(counts)))
        if not fh.is_pinned():
            fh = fh.pin_memory()
        R = fh.shape[0]
        # one plan: RHS groups with a shared copy pipeline (DS_HOST_GROUPS=1,
        # ds_ddm_apply_host_groups) measured 5.39 vs 5.05 ms on config 2 --
        # the PCIe phases gate both groups alike (tools/host_groups_probe.py)
        dp = device_plan(partition, operators, cache, plan, R,
                         grouped=os.environ.get("DS_HOST_GROUPS", "0") == "1")
        uh = torch.empty(fh.shape, dtype=torch.complex128, pin_memory=True)
        dp.apply_host(fh, uh)
        reports = _reports(dp, R, plan, partition, record_events, record_transfers)
        wall = time.perf_counter() - t0
        for rep in reports:
            rep.wall_time = wall
        values = uh.reshape((R,) + counts) if batched else uh.reshape(counts)
        return ComplexField(partition.grid, values), (reports if batched else reports[0])
    if shape[1:] == counts and shape[0] == 0:
        return _empty_batch(f, partition), []
    fdev, kind, batched = _engine.to_device_batch(f, counts)
    R = fdev.shape[0]
    chunk = 256
    us, parts_all, reports = [], [], []
    for r0 in range(0, R, chunk):
        fr = fdev[r0:r0 + chunk].reshape(min(chunk, R - r0), -1)
        dp = device_plan(partition, operators, cache, plan, fr.shape[0],
                         pipelined=None if not collect_partials else False,
                         grouped=not collect_partials)
        u, parts = dp.apply(fr, collect_partials=collect_partials)
        us.append(u)
        parts_all.append(parts)
        reports += _reports(dp, fr.shape[0], plan, partition, record_events, record_transfers)
    import torch

    u = torch.cat(us, 0).reshape((R,) + counts) if len(us) > 1 else us[0].reshape((R,) + counts)
    torch.cuda.current_stream().synchronize()
    wall = time.perf_counter() - t0
    for r, rep in enumerate(reports):
        rep.wall_time = wall
        if collect_partials:
            chunk_i, rr = divmod(r, chunk)
            rep.partials = [_engine.from_device_batch(p[rr:rr + 1].reshape((1,) + counts), kind, False)
                            for p in parts_all[chunk_i]]
    values = _engine.from_device_batch(u, kind, batched)
    field_out = ComplexField(partition.grid, values)
    return field_out, (reports if batched else reports[0])


def additive_ddm_solve(f, partition: Partition, operators: dict,
                       cache: FactorizationCache | None = None, *, warn_collar: bool = True):
    """The additive overlapping DDM baseline (all subdomains at every step),
    `additive_ddm_solve` (ddm.py:294-349), batched over RHS, on the same
    kernels as the diagonal sweep (one device "sweep" per step; see
    `_engine.DevicePlan`).  Returns (ComplexField, DdmReport or [DdmReport])."""
    from . import _engine

    t0 = time.perf_counter()
    counts = partition.grid.counts
    shape = tuple(f.shape)
    if shape != counts and shape[1:] != counts:
        raise ConfigurationError("source shape does not match the grid")
    if cache is None:
        cache = FactorizationCache()
    if not isinstance(cache, FactorizationCache):
        raise ConfigurationError("cache must be a paper_2002_05327_b200 FactorizationCache")
    if warn_collar:
        _warn_collar(f, partition)
    if shape[1:] == counts and shape[0] == 0:
        return _empty_batch(f, partition), []
    fdev, kind, batched = _engine.to_device_batch(f, counts)
    R = fdev.shape[0]
    chunk = 256
    us, reports = [], []
    for r0 in range(0, R, chunk):
        fr = fdev[r0:r0 + chunk].reshape(min(chunk, R - r0), -1)
        dp = device_plan(partition, operators, cache, None, fr.shape[0], schedule="additive")
        u, _ = dp.apply(fr)
        us.append(u)
        ctr = dp.counters(fr.shape[0])
        for r in range(fr.shape[0]):
            rep = DdmReport(solves=dp.nsweeps * dp.nsub, nonzero_solves=int(ctr["nonzero"][r]),
                            discarded_sources=int(ctr["discarded"][r]))
            vnz = ctr["visit_nonzero"][:, :, r]
            for s, idx in enumerate(dp.subs):
                steps = np.nonzero(vnz[:, s])[0]
                if steps.size:
                    rep.first_nonzero_step[idx] = int(steps[0]) + 1
            reports.append(rep)
    import torch

    u = torch.cat(us, 0).reshape((R,) + counts) if len(us) > 1 else us[0].reshape((R,) + counts)
    torch.cuda.current_stream().synchronize()
    wall = time.perf_counter() - t0
    for rep in reports:
        rep.wall_time = wall
    values = _engine.from_device_batch(u, kind, batched)
    return ComplexField(partition.grid, values), (reports if batched else reports[0])


def _empty_batch(f, partition: Partition) -> ComplexField:
    """The result of an empty batch [0, *counts]: an empty field of the
    input's kind (an empty RHS shard of a multi-rank run, distributed.py)."""
    shape = (0,) + tuple(partition.grid.counts)
    if hasattr(f, "detach"):
        import torch

        return ComplexField(partition.grid, torch.zeros(shape, dtype=torch.complex128,
                                                        device=f.device))
    return ComplexField(partition.grid, np.zeros(shape, dtype=np.complex128))


def _reports(dp, nrhs: int, plan: SweepPlan, partition: Partition, record_events: bool,
             record_transfers: bool):
    ctr = dp.counters(nrhs)
    dim = partition.dim
    solves = len(plan.directions) * dp.nsub
    reports = []
    for r in range(nrhs):
        rep = DdmReport(solves=solves, nonzero_solves=int(ctr["nonzero"][r]),
                        discarded_sources=int(ctr["discarded"][r]),
                        events=[] if record_events else None,
                        transfer_records=[] if record_transfers else None)
        if record_events or record_transfers:
            for w in range(dp.nsweeps):
                for t in range(dp.nsteps):
                    b, e = dp.step_off[w * (dp.nsteps + 1) + t], dp.step_off[w * (dp.nsteps + 1) + t + 1]
                    for s in dp.visit_sub[w * dp.nsub + b: w * dp.nsub + e]:
                        nz = bool(ctr["visit_nonzero"][w, s, r])
                        idx = dp.subs[s]
                        if record_events:
                            rep.events.append({
                                "sweep": w + 1, "step": t + 1, "subdomain": list(idx),
                                "sources_consumed": int(ctr["visit_consumed"][w, s, r]),
                                "sources_emitted": int(ctr["visit_emitted"][w, s, r]),
                                "nonzero": nz})
                        if record_transfers and nz:
                            cuts = cut_mask_to_set(int(ctr["visit_cut"][w, s, r]), dim)
                            for k, dvec in enumerate(dp.dirs):
                                if not emits(dvec, cuts) or dp.geoms[(s, k)] is None:
                                    continue
                                use = int(dp.xfer_use[w, s, k])
                                target = tuple(i + c for i, c in zip(idx, dvec))
                                rep.transfer_records.append(
                                    (w + 1, dvec, idx, target, use if use else "discarded"))
        reports.append(rep)
    return reports


def octant_exactness_check(partials, reference, partition: Partition, origin, plan=None):
    """Per-sweep relative errors of the partial sums on their octants (test
    helper, ddm.py:352-378)."""
    plan = plan or SweepPlan.default(partition.dim)
    out = []
    for sweep, direction in enumerate(plan.directions, 1):
        region = octant_region(direction, origin, partition.counts)
        mask = np.zeros(partition.grid.counts, dtype=bool)
        for index in region.indices:
            mask[partition.box(index).slices()] = True
        part = np.asarray(partials[sweep - 1])
        ref_norm = np.linalg.norm(reference[mask]) if mask.any() else 0.0
        rel = 0.0 if ref_norm == 0.0 else float(
            np.linalg.norm(part[mask] - reference[mask]) / ref_norm)
        out.append({"sweep": sweep, "direction": direction,
                    "subdomains": len(region.indices), "relative_error": rel})
    return out
