"""Subdomain-sharded diagonal sweep (SURVEY §8(e) spatial alternative, §8(f)
rank 1): each rank owns a block of subdomains, factorizes only their
operators and runs only their visits of the global launch schedule.

Data path (no separate exchange step): payload slots live on the rank that
owns their target; a rank's transfer kernel (K4) writes payloads and arrival
flags of remote targets straight into the owner's memory through peer
pointers (NVLink P2P / CUDA IPC mappings), the paper's point-to-point band
transfer (`PAPER.md:1290-1294`) fused into the producing kernel.  Every slot
has exactly one source subdomain, so its writers are on one rank, and the
consuming assembly (K6) zeroes it in place.  Ordering: every rank initialises
its flags, then for each launch l every rank runs launch l, with a cross-rank
barrier between launches; the sweep's u is the sum of the ranks' u.

Two runners share that protocol:
* `ShardedSweep` -- virtual ranks in one process on one device (one plan per
  rank, launches issued rank after rank on one stream, so no kernel ever
  waits on another).  It exercises the whole sharded data path on one GPU and
  is what the tests check against the unsharded sweep.
* `DistributedShardedSweep` -- one process per GPU (torch.distributed, NCCL):
  peers' slot, flag and barrier allocations are mapped with CUDA IPC handles
  exchanged once through the process group; the barrier between launches is
  a device-side flag barrier in peer memory (`DeviceBarrier`,
  ds_barrier_wait: one single-warp kernel per launch, no host round trip
  and no collective); NCCL only sums u at the end.  barrier="nccl" keeps the
  former stream-ordered all-reduce on a token.
"""
from __future__ import annotations

import numpy as np

from . import _engine
from .ddm import SweepPlan
from .errors import ConfigurationError


def block_owners(partition, nranks: int, axis: int = 0):
    """owner[s] for the subdomains in `partition.subdomains()` order: contiguous
    blocks of subdomain rows along `axis` (neighbouring ranks exchange bands
    only across one block face)."""
    n = partition.counts[axis]
    if not 1 <= nranks <= n:
        raise ConfigurationError(f"nranks must be in [1, {n}] for a block split along axis {axis}")
    return [((idx[axis] - 1) * nranks) // n for idx in partition.subdomains()]


def _merge_counters(parts):
    out = {}
    for k in parts[0]:
        if k == "visit_cut":
            acc = parts[0][k].copy()
            for p in parts[1:]:
                acc |= p[k]
        else:
            acc = sum(p[k] for p in parts)
        out[k] = acc
    return out


class ShardedSweep:
    """Virtual ranks on one device (see the module docstring)."""

    def __init__(self, partition, operators, nranks: int, nrhs_max: int, caches=None,
                 plan: SweepPlan | None = None, pipelined: bool = True, owner=None):
        plan = plan or SweepPlan.default(partition.dim)
        self.partition = partition
        self.nranks = nranks
        self.owner = list(owner) if owner is not None else block_owners(partition, nranks)
        if caches is None:
            from .subdomain import FactorizationCache
            caches = [FactorizationCache() for _ in range(nranks)]
        self.plans = [
            _engine.DevicePlan(partition, operators, caches[r], plan.directions, nrhs_max,
                               pipelined=pipelined, shard=(nranks, r, self.owner))
            for r in range(nranks)]
        infos = [p.shard_info() for p in self.plans]
        for p in self.plans:
            p.set_peers([i[0] for i in infos], [i[2] for i in infos])
        self.nlaunch = self.plans[0].nlaunch()
        if any(p.nlaunch() != self.nlaunch for p in self.plans):
            raise ConfigurationError("ranks disagree on the launch schedule")
        self.nnodes = self.plans[0].nnodes
        self._bufs = {}

    def apply(self, f):
        """f: [R, N] complex128 CUDA tensor (RHS-outer) -> u [R, N]."""
        import torch

        lib, ctx = _engine.context()
        R, n = f.shape[0], self.nnodes
        if R not in self._bufs:
            fmin = torch.empty((n, R), dtype=torch.complex128, device=f.device)
            self._bufs[R] = (fmin, [torch.empty_like(fmin) for _ in range(self.nranks)])
        fmin, umins = self._bufs[R]
        _engine.N.check(lib.ds_layout_to_minor(ctx, n, R, f.data_ptr(), fmin.data_ptr()))
        for p, um in zip(self.plans, umins):  # every rank's flags zeroed before any peer write
            p.apply_range(fmin, um, R, 0, 0, 1)
        for l in range(self.nlaunch):
            for p, um in zip(self.plans, umins):
                p.apply_range(fmin, um, R, l, l + 1, 0)
        for p, um in zip(self.plans, umins):
            p.apply_range(fmin, um, R, self.nlaunch, self.nlaunch, 2)
        usum = umins[0].clone()
        for um in umins[1:]:
            usum += um
        u = torch.empty((R, n), dtype=torch.complex128, device=f.device)
        _engine.N.check(lib.ds_layout_to_outer(ctx, n, R, usum.data_ptr(), u.data_ptr()))
        return u

    def counters(self, nrhs: int):
        return _merge_counters([p.counters(nrhs) for p in self.plans])


class DeviceBarrier:
    """Rank `rank` of an `nranks` device-side barrier (ds_barrier_*): its
    arrival array lives in this rank's memory; `set_peers` takes every
    rank's array (local, peer or IPC-mapped); `wait()` enqueues the barrier
    on the current stream."""

    def __init__(self, nranks: int, rank: int):
        import ctypes as C
        import weakref

        lib, ctx = _engine.context()
        out = C.c_void_p()
        _engine.N.check(lib.ds_barrier_create(ctx, nranks, rank, C.byref(out)), "ds_barrier_create")
        self.handle = out
        self.nranks, self.rank = nranks, rank
        self._finalizer = weakref.finalize(self, lib.ds_barrier_destroy, out)

    def arrive_ptr(self) -> int:
        import ctypes as C

        p = C.c_void_p()
        _engine.N.check(_engine.N.load_library().ds_barrier_info(self.handle, C.byref(p), None))
        return p.value

    def set_peers(self, ptrs):
        import ctypes as C

        arr = (C.c_void_p * len(ptrs))(*ptrs)
        _engine.N.check(_engine.N.load_library().ds_barrier_set_peers(self.handle, len(ptrs), arr),
                        "ds_barrier_set_peers")

    def wait(self):
        lib, ctx = _engine.context()
        _engine.N.check(lib.ds_barrier_wait(ctx, self.handle), "ds_barrier_wait")

    @property
    def generation(self) -> int:
        return int(_engine.N.load_library().ds_barrier_generation(self.handle))


class DistributedShardedSweep:
    """One process per GPU (torch.distributed with the NCCL backend; see the
    module docstring).  Each rank holds only its owned factorizations; the
    returned u (on every rank) is the all-reduced sum."""

    def __init__(self, partition, operators, nrhs_max: int, group=None, cache=None,
                 plan: SweepPlan | None = None, pipelined: bool = True, barrier: str = "device"):
        import torch.distributed as dist

        from .subdomain import FactorizationCache

        self.dist, self.group = dist, group
        self.nranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        plan = plan or SweepPlan.default(partition.dim)
        self.owner = block_owners(partition, self.nranks)
        self.plan = _engine.DevicePlan(partition, operators, cache or FactorizationCache(),
                                       plan.directions, nrhs_max, pipelined=pipelined,
                                       shard=(self.nranks, self.rank, self.owner))
        slot, _, flags, _ = self.plan.shard_info()
        if barrier not in ("device", "nccl"):
            raise ConfigurationError(f"unknown barrier {barrier!r}")
        self.barrier = DeviceBarrier(self.nranks, self.rank) if barrier == "device" else None
        mine = [_ipc_handle(slot), _ipc_handle(flags)]
        if self.barrier is not None:
            mine.append(_ipc_handle(self.barrier.arrive_ptr()))
        handles = [None] * self.nranks
        dist.all_gather_object(handles, tuple(mine), group=group)
        slots = [slot if r == self.rank else _ipc_open(handles[r][0]) for r in range(self.nranks)]
        flagp = [flags if r == self.rank else _ipc_open(handles[r][1]) for r in range(self.nranks)]
        self.plan.set_peers(slots, flagp)
        if self.barrier is not None:
            self.barrier.set_peers([self.barrier.arrive_ptr() if r == self.rank else _ipc_open(handles[r][2])
                                    for r in range(self.nranks)])
        self.nlaunch = self.plan.nlaunch()
        self.nnodes = self.plan.nnodes
        self._bufs = {}

    def apply(self, f):
        import torch

        lib, ctx = _engine.context()
        R, n = f.shape[0], self.nnodes
        if R not in self._bufs:
            fmin = torch.empty((n, R), dtype=torch.complex128, device=f.device)
            self._bufs[R] = (fmin, torch.empty_like(fmin))
        fmin, umin = self._bufs[R]
        _engine.N.check(lib.ds_layout_to_minor(ctx, n, R, f.data_ptr(), fmin.data_ptr()))
        run_protocol(self.plan, fmin, umin, R, self.dist, self.group, device=f.device,
                     barrier=self.barrier.wait if self.barrier is not None else None)
        u = torch.empty((R, n), dtype=torch.complex128, device=f.device)
        _engine.N.check(lib.ds_layout_to_outer(ctx, n, R, umin.data_ptr(), u.data_ptr()))
        return u


def run_protocol(plan, fmin, umin, nrhs: int, dist, group=None, device="cuda", barrier=None):
    """One sharded application on this rank: initialise (zero u and flags),
    barrier (no peer writes into flags not yet zeroed), every launch followed
    by a barrier (a launch's consumers may sit on any rank), finalise, then
    sum u over the ranks.  `barrier` (a callable enqueuing a device barrier
    on the current stream, DeviceBarrier.wait) or, if None, an all-reduce on
    a token queued on the current stream; neither syncs the host."""
    import torch

    if barrier is None:
        def barrier():
            tok = torch.zeros(1, device=device)
            dist.all_reduce(tok, group=group)

    nl = plan.nlaunch()
    plan.apply_range(fmin, umin, nrhs, 0, 0, 1)
    barrier()
    for l in range(nl):
        plan.apply_range(fmin, umin, nrhs, l, l + 1, 0)
        barrier()
    plan.apply_range(fmin, umin, nrhs, nl, nl, 2)
    dist.all_reduce(umin, group=group)


def _ipc_handle(ptr: int) -> bytes:
    from cuda.bindings import runtime as rt

    err, h = rt.cudaIpcGetMemHandle(ptr)
    if err != rt.cudaError_t.cudaSuccess:
        raise ConfigurationError(f"cudaIpcGetMemHandle: {err}")
    return bytes(h.reserved)


def _ipc_open(handle: bytes) -> int:
    from cuda.bindings import runtime as rt

    h = rt.cudaIpcMemHandle_t()
    h.reserved = handle
    err, ptr = rt.cudaIpcOpenMemHandle(h, rt.cudaIpcMemLazyEnablePeerAccess)
    if err != rt.cudaError_t.cudaSuccess:
        raise ConfigurationError(f"cudaIpcOpenMemHandle: {err}")
    return int(ptr)
