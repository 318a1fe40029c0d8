"""GPU runtime glue between the reference-shaped Python API and the C-ABI.

PyTorch is used only as plumbing: CUDA device memory, the current stream
and host<->device copies.  All arithmetic of the hot path runs in the
hand-written kernels of `libdiagsweep_b200.so`; when no CUDA device or no
library is present the calls raise `SolverError` (no CPU fallback).

Layouts: user-facing batches are RHS-outer `[R, *shape]` (the reference's
array layout with a leading batch axis); the sweep engine works RHS-minor
internally and converts with the `ds_layout_*` kernels at its boundary.
"""

from __future__ import annotations

import ctypes as C
import itertools
import math
import os
import weakref

import numpy as np

from . import _native as N
from .errors import ConfigurationError, SolverError

try:  # torch is plumbing only; imported lazily-safe for CPU-only test runs
    import torch
except Exception:  # pragma: no cover
    torch = None

_CTX: dict = {}


def _require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise SolverError(
            "no CUDA device: the diagsweep_b200 hot path runs only on the GPU "
            "(there is no CPU fallback)")


def launch_count() -> int:
    """Kernels the native library has launched on this device's context."""
    lib, ctx = context()
    return int(lib.ds_ctx_launches(ctx))


def context():
    """(lib, ctx) bound to torch's current device and stream."""
    _require_cuda()
    lib = N.load_library()
    dev = torch.cuda.current_device()
    h = _CTX.get(dev)
    if h is None:
        out = C.c_void_p()
        N.check(lib.ds_ctx_create(dev, None, C.byref(out)), "ds_ctx_create")
        h = out
        _CTX[dev] = h
    N.check(lib.ds_ctx_set_stream(h, C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return lib, h


def set_option(name: str, value: int) -> int:
    """Set a variant / tuning option of this device's native context
    (ds_ctx_set_option); returns the previous value.  Plans capture CUDA
    graphs with the options in force when they were recorded."""
    lib, ctx = context()
    old = C.c_int32()
    N.check(lib.ds_ctx_get_option(ctx, name.encode(), C.byref(old)), "ds_ctx_get_option")
    N.check(lib.ds_ctx_set_option(ctx, name.encode(), int(value)), "ds_ctx_set_option")
    return old.value


def executed_work(reset: bool = False) -> int:
    """Complex multiply-adds the modal transforms executed on this device's
    context while the option "count_work" was 1 (ds_ctx_work); measurement
    only (bench.py's roofline numerator)."""
    lib, ctx = context()
    v = C.c_int64()
    N.check(lib.ds_ctx_work(ctx, C.byref(v), 1 if reset else 0), "ds_ctx_work")
    return int(v.value)


def get_option(name: str) -> int:
    lib, ctx = context()
    v = C.c_int32()
    N.check(lib.ds_ctx_get_option(ctx, name.encode(), C.byref(v)), "ds_ctx_get_option")
    return v.value


# ----------------------------------------------------------------- tensors

def is_pinned_host(v) -> bool:
    """A page-locked CPU torch tensor (the zero-staging host path)."""
    return hasattr(v, "detach") and not v.is_cuda and v.is_pinned()


def to_device_batch(v, shape):
    """-> (tensor [R, *shape] complex128 contiguous on the GPU, kind, batched)."""
    _require_cuda()
    kind = ("torch" if v.is_cuda else "torch_cpu") if hasattr(v, "detach") else "numpy"
    vshape = tuple(v.shape)
    if vshape == tuple(shape):
        batched = False
    elif vshape[1:] == tuple(shape):
        batched = True
    else:
        raise ConfigurationError(f"field shape {vshape} does not match window {tuple(shape)}")
    if kind == "numpy":
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.complex128))
        t = t.to("cuda", non_blocking=False)
    else:
        t = v.detach()
        if t.dtype != torch.complex128:
            t = t.to(torch.complex128)
        if not t.is_cuda:
            t = t.to("cuda", non_blocking=t.is_pinned())
        t = t.contiguous()
    if not batched:
        t = t.reshape((1,) + tuple(shape))
    return t, kind, batched


def from_device_batch(t, kind, batched):
    if not batched:
        t = t[0]
    if kind == "numpy":
        return t.cpu().numpy()
    if kind == "torch_cpu":
        # host result in pinned memory (one DMA, no pageable staging copy)
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    return t


# --------------------------------------------------------------- operators

KINDS = {"const": 0, "axis": 1, "full": 2}


def op_couplings(op):
    """(c_lo, c_hi) per axis through the reference's public surface
    (`DiscreteOperator.axis_coefficients`, pml.py:95-102); our own operator
    class caches them as `.couplings`."""
    cp = getattr(op, "couplings", None)
    if cp is not None:
        return cp
    return [op.axis_coefficients(a) for a in range(op.grid.dim)]


def op_kappa2(op):
    """(kind code, axis, flat float64 array) of kappa^2 from the reference's
    `kappa2_kind` / `kappa2` fields ('const' float, 'axis' (axis, values),
    'full' ndarray; pml.py:75-84)."""
    kind = op.kappa2_kind
    if kind == "const":
        return KINDS[kind], -1, np.array([float(op.kappa2)])
    if kind == "axis":
        axis, values = op.kappa2
        return KINDS[kind], int(axis), np.ascontiguousarray(values, dtype=np.float64)
    return KINDS[kind], -1, np.ascontiguousarray(op.kappa2, dtype=np.float64).ravel()


class DeviceOperator:
    """Device copy of one DiscreteOperator's couplings and kappa^2.  Reads
    only the reference's public operator surface (window, grid,
    axis_coefficients, kappa2_kind, kappa2), so the reference's own
    `DiscreteOperator` objects work too."""

    def __init__(self, op):
        lib, ctx = context()
        keep = []
        desc = N.OpDesc()
        dim = op.grid.dim
        desc.dim = dim
        for a, (lo, hi) in enumerate(op_couplings(op)):
            lo = np.ascontiguousarray(lo, dtype=np.complex128)
            hi = np.ascontiguousarray(hi, dtype=np.complex128)
            keep += [lo, hi]
            desc.shape[a] = op.window.shape[a]
            desc.c_lo[a] = lo.ctypes.data
            desc.c_hi[a] = hi.ctypes.data
        kind, axis, k2 = op_kappa2(op)
        keep.append(k2)
        desc.kappa2_kind = kind
        desc.kappa2_axis = axis
        desc.kappa2 = k2.ctypes.data
        out = C.c_void_p()
        N.check(lib.ds_op_create(ctx, C.byref(desc), C.byref(out)), "ds_op_create")
        self.handle = out
        self.shape = tuple(op.window.shape)
        self._finalizer = weakref.finalize(self, lib.ds_op_destroy, out)


# device operators of foreign (reference) operator objects, content-keyed by
# fingerprint + shape (the reference's dataclass is unhashable and has no
# slot for a device handle); entries live as long as a factorization or plan
# holds the DeviceOperator
_FOREIGN_DEVOPS: "weakref.WeakValueDictionary" = weakref.WeakValueDictionary()


def device_operator(op) -> DeviceOperator:
    if hasattr(op, "_device"):
        if op._device is None:
            op._device = DeviceOperator(op)
        return op._device
    key = (op.fingerprint, tuple(op.window.shape), torch.cuda.current_device())
    dop = _FOREIGN_DEVOPS.get(key)
    if dop is None:
        dop = DeviceOperator(op)
        _FOREIGN_DEVOPS[key] = dop
    return dop


def apply_operator(op, v, region):
    lib, ctx = context()
    dop = device_operator(op)
    t, kind, batched = to_device_batch(v, region.shape)
    out = torch.empty_like(t)
    lo = np.array([r - w for r, w in zip(region.lo, op.window.lo)] + [0] * (3 - op.dim),
                  dtype=np.int32)
    sh = np.array(list(region.shape) + [1] * (3 - op.dim), dtype=np.int32)
    N.check(lib.ds_op_apply(ctx, dop.handle, t.data_ptr(), out.data_ptr(), t.shape[0],
                            lo.ctypes.data_as(N.P_i32), sh.ctypes.data_as(N.P_i32), 1),
            "ds_op_apply")
    return from_device_batch(out, kind, batched)


# ------------------------------------------------------------ factorization

def block_axis_of(shape) -> int:
    """Block axis of the layout: the longest window axis, first on ties."""
    return int(np.argmax(np.asarray(shape)))


def axis_tridiagonal(op, axis: int) -> np.ndarray:
    """Dense 1D operator of `axis` (pml.py couplings; kappa^2 folded in
    when it varies along this axis) -- the factor the reference's
    SeparableFactorization triangularizes (subdomain.py:52-63)."""
    lo, hi = op_couplings(op)[axis]
    n = len(lo)
    T = np.zeros((n, n), dtype=np.complex128)
    i = np.arange(n)
    T[i, i] = -(lo + hi)
    T[i[1:], i[1:] - 1] = lo[1:]
    T[i[:-1], i[:-1] + 1] = hi[:-1]
    if op.kappa2_kind == "axis" and op.kappa2[0] == axis:
        T[i, i] += np.asarray(op.kappa2[1], dtype=np.float64)
    return T


_EIG_CACHE: dict = {}


def _axis_eig(T: np.ndarray):
    """(V, V^{-1}, lambda, quality) of one 1D matrix, memoised on its bytes
    (windows of a partition share most of their per-axis operators).
    quality = (cond_2(V), ||T V - V diag(lambda)||_F / (||T||_F ||V||_F),
    ||V^{-1} V - I||_F): the numbers the modal factorization's guard checks."""
    key = T.tobytes()
    hit = _EIG_CACHE.get(key)
    if hit is None:
        lam, V = np.linalg.eig(T)
        W = np.linalg.inv(V)
        sv = np.linalg.svd(V, compute_uv=False)
        cond = float(sv[0] / sv[-1]) if sv[-1] > 0 else math.inf
        nT, nV = np.linalg.norm(T), np.linalg.norm(V)
        res = float(np.linalg.norm(T @ V - V * lam) / (nT * nV)) if nT and nV else math.inf
        inv_err = float(np.linalg.norm(W @ V - np.eye(len(lam))))
        if not np.all(np.isfinite(W)):
            cond = inv_err = math.inf
        hit = (np.ascontiguousarray(V, dtype=np.complex128),
               np.ascontiguousarray(W, dtype=np.complex128),
               np.ascontiguousarray(lam, dtype=np.complex128),
               (cond, res, inv_err))
        if len(_EIG_CACHE) > 4096:
            _EIG_CACHE.clear()
        _EIG_CACHE[key] = hit
    return hit


def modal_decomposition(op):
    """Eigen-decompositions T_a = V diag(lambda) V^{-1} of the in-slab axes
    (LAPACK zgeev through NumPy; n_a <= a few hundred, O(n_a^3) each).
    Returns (block_axis, [(V, V^{-1}, lambda, quality), ...]) in in-slab axis
    order."""
    ba = block_axis_of(op.window.shape)
    return ba, [_axis_eig(axis_tridiagonal(op, a)) for a in range(op.dim) if a != ba]


# Guard of the modal factorization.  The eigenbasis V_a is not unitary (the
# reference's Schur basis is), so the mode-wise solve loses about
# log10(cond(V_a)) digits: configs 1/2/4 have cond(V) = 3e3 / 2e4 / 60 and
# solve to <= 1.2e-12 of the Schur/Sylvester oracle.  Above these limits the
# operator is factored by the block LU instead (same kernels as raster media).
MODAL_COND_MAX = 1e6
MODAL_RESIDUAL_MAX = 1e-12
MODAL_INVERSE_MAX = 1e-9


def modal_guard(op, cond_max: float = MODAL_COND_MAX):
    """(ok, reason, decomposition): whether the modal factorization of `op`
    is well conditioned enough to keep the 1e-10 parity bar.  cond_max =
    inf disables the guard (measurements of the unguarded modal path)."""
    ba, axes = modal_decomposition(op)
    if cond_max == math.inf:
        return True, "", (ba, axes)
    for a, (_, _, _, (cond, res, inv_err)) in enumerate(axes):
        if not cond <= cond_max:
            return False, f"in-slab axis {a}: cond(V) {cond:.3g} > {cond_max:.3g}", (ba, axes)
        if not res <= MODAL_RESIDUAL_MAX:
            return False, f"in-slab axis {a}: eigen-residual {res:.3g}", (ba, axes)
        if not inv_err <= MODAL_INVERSE_MAX:
            return False, f"in-slab axis {a}: ||V^-1 V - I|| {inv_err:.3g}", (ba, axes)
    return True, "", (ba, axes)


class FactorSet:
    """One ds_fact handle holding the factors of several operators: the
    block-tridiagonal LU (K2, any operator) or, with `modal`, the modal
    factorization of separable operators (K2m, ds_modal.cu)."""

    def __init__(self, ops, modal: bool = False, decomps=None):
        lib, ctx = context()
        dops = [device_operator(op) for op in ops]
        arr = (C.c_void_p * len(ops))(*[d.handle.value for d in dops])
        out = C.c_void_p()
        self.modal = modal
        if modal:
            descs = (N.ModalDesc * len(ops))()
            keep = []
            for i, op in enumerate(ops):
                ba, axes = decomps[i] if decomps is not None else modal_decomposition(op)
                descs[i].block_axis = ba
                descs[i].naxes = len(axes)
                for a, (V, W, lam, _q) in enumerate(axes):
                    keep += [V, W, lam]
                    descs[i].v[a] = V.ctypes.data
                    descs[i].vinv[a] = W.ctypes.data
                    descs[i].lambda_[a] = lam.ctypes.data
            N.check(lib.ds_fact_create_modal(ctx, arr, len(ops), descs, C.byref(out)),
                    "ds_fact_create_modal")
            del keep
        else:
            N.check(lib.ds_fact_create(ctx, arr, len(ops), C.byref(out)), "ds_fact_create")
        self.handle = out
        self.n = len(ops)
        self._dops = dops  # device operators must outlive the factors
        self._finalizer = weakref.finalize(self, lib.ds_fact_destroy, out)

    def info(self, i):
        lib = N.load_library()
        ba, nb, m = C.c_int32(), C.c_int32(), C.c_int32()
        nbytes = C.c_int64()
        N.check(lib.ds_fact_info(self.handle, i, C.byref(ba), C.byref(nb), C.byref(m),
                                 C.byref(nbytes)))
        return ba.value, nb.value, m.value, nbytes.value


class FactorPool:
    """Out-of-core block-LU factors (ds_fact_create_pool): the layouts of
    `ops` and `nslots` device slots of the largest operator's factor size;
    `load(i, slot)` factors operator i into a slot (K2b), evicting its
    previous owner.  For factor sets larger than HBM (config 5: 64 raster
    windows, 638 GB of dense block inverses)."""

    modal = False

    def __init__(self, ops, nslots: int):
        lib, ctx = context()
        self._dops = [device_operator(op) for op in ops]
        arr = (C.c_void_p * len(ops))(*[d.handle.value for d in self._dops])
        out = C.c_void_p()
        N.check(lib.ds_fact_create_pool(ctx, arr, len(ops), int(nslots), C.byref(out)),
                "ds_fact_create_pool")
        self.handle = out
        self.n = len(ops)
        self.nslots = int(nslots)
        self._finalizer = weakref.finalize(self, lib.ds_fact_destroy, out)

    def load(self, i: int, slot: int):
        lib, ctx = context()
        N.check(lib.ds_fact_pool_load(ctx, self.handle, int(i), int(slot)), "ds_fact_pool_load")

    def load_many(self, pairs):
        """[(operator, slot), ...] factored in one batch (chains advance together)."""
        if not pairs:
            return
        lib, ctx = context()
        idx = np.asarray([p[0] for p in pairs], np.int32)
        slots = np.asarray([p[1] for p in pairs], np.int32)
        N.check(lib.ds_fact_pool_load_many(ctx, self.handle, len(pairs), idx.ctypes.data_as(N.P_i32),
                                           slots.ctypes.data_as(N.P_i32)), "ds_fact_pool_load_many")

    def state(self):
        """(slot owners, slot bytes, factorizations run)."""
        lib = N.load_library()
        ns, sb, loads = C.c_int32(), C.c_int64(), C.c_int64()
        owners = (C.c_int32 * self.nslots)()
        N.check(lib.ds_fact_pool_state(self.handle, C.byref(ns), C.byref(sb), owners, C.byref(loads)))
        return list(owners), sb.value, loads.value

    def info(self, i):
        lib = N.load_library()
        ba, nb, m = C.c_int32(), C.c_int32(), C.c_int32()
        nbytes = C.c_int64()
        N.check(lib.ds_fact_info(self.handle, i, C.byref(ba), C.byref(nb), C.byref(m),
                                 C.byref(nbytes)))
        return ba.value, nb.value, m.value, nbytes.value


def block_lu_bytes(shape) -> int:
    """Dense block-inverse bytes of the block LU of a window (n_b m^2 complex)."""
    nb = max(shape)
    m = int(np.prod(shape)) // nb
    return nb * m * m * 16


def belady_slots(launches, nslots: int):
    """Static slot assignment for pooled factors over a launch schedule:
    every visit of a launch gets a distinct slot holding its subdomain's
    factors; a subdomain not resident is loaded into the slot whose owner is
    next used furthest in the future (Belady's optimal replacement, known
    schedule).  Returns ({(sweep, sub): slot}, per-launch [(sub, slot)]
    loads, total loads)."""
    order = [sv for L in launches for (_, sv) in L]
    pos_of = {}
    for p in range(len(order) - 1, -1, -1):
        pos_of.setdefault(order[p], []).append(p)  # reversed positions per subdomain
    owner = [None] * nslots
    slot_of = {}
    visit_slot, loads = {}, []
    p = 0
    for L in launches:
        need = {sv for (_, sv) in L}
        if len(need) > nslots:
            raise ConfigurationError("factor pool: a launch needs more slots than the pool has")
        here = []
        for (w, sv) in L:
            stack = pos_of[sv]
            while stack and stack[-1] < p:
                stack.pop()
        for (w, sv) in L:
            if sv not in slot_of:
                free = [c for c in range(nslots) if owner[c] is None]
                if free:
                    c = free[0]
                else:
                    def next_use(c):
                        st = pos_of[owner[c]]
                        while st and st[-1] < p:
                            st.pop()
                        return st[-1] if st else math.inf
                    cands = [c for c in range(nslots) if owner[c] not in need]
                    c = max(cands, key=lambda c: (next_use(c), -c))
                    del slot_of[owner[c]]
                owner[c] = sv
                slot_of[sv] = c
                here.append((sv, c))
            visit_slot[(w, sv)] = slot_of[sv]
        loads.append(here)
        p += len(L)
    return visit_slot, loads, sum(len(h) for h in loads)


def fact_solve(fset: FactorSet, index: int, shape, rhs):
    lib, ctx = context()
    t, kind, batched = to_device_batch(rhs, shape)
    R = t.shape[0]
    W = int(np.prod(shape))
    tmin = torch.empty((W, R), dtype=torch.complex128, device=t.device)
    N.check(lib.ds_layout_to_minor(ctx, W, R, t.data_ptr(), tmin.data_ptr()))
    xmin = torch.empty_like(tmin)
    N.check(lib.ds_fact_solve(ctx, fset.handle, index, tmin.data_ptr(), xmin.data_ptr(), R),
            "ds_fact_solve")
    x = torch.empty_like(t)
    N.check(lib.ds_layout_to_outer(ctx, W, R, xmin.data_ptr(), x.data_ptr()))
    return from_device_batch(x, kind, batched)


# -------------------------------------------------------------- sweep plan

def source_directions(dim: int):
    return tuple(d for d in itertools.product((-1, 0, 1), repeat=dim) if any(d))


def _pad3(t, fill=0):
    t = list(t)
    return t + [fill] * (3 - len(t))


def launch_schedule(nsweeps: int, nsub: int, order, xfer_use, dirs, sub_index, in_range,
                    cap: int, resident: int = 0):
    """List-schedule the (sweep, subdomain) visits of one application.

    `order` is the sequential visit order (sweep by sweep, step by step); a
    visit depends on every source visit routed to it (xfer_use; this covers
    its step predecessors) and on the previous writer of each payload slot
    it writes (slots accumulate non-atomically, and the fixed writer order
    keeps the sums deterministic).  Ready visits are taken longest remaining
    path first, at most `cap` per launch.  Returns a list of launches, each a
    list of (sweep 0-based, subdomain) in launch order.

    resident > 0 (out-of-core factor pools): ready visits whose subdomain is
    among the `resident` most recently scheduled ones go first -- their
    factors are still in a pool slot.  Config 5 (64 windows, 10 slots, one
    visit per launch): 354 factorizations per application instead of 384
    (Belady replacement over either order)."""
    pos = {v: i for i, v in enumerate(order)}
    deps = {v: set() for v in order}
    last_writer = {}
    for (w, s) in order:
        for k, d in enumerate(dirs):
            use = int(xfer_use[w, s, k])
            if use < 1:
                continue
            t = sub_index(s, d)
            deps[(use - 1, t)].add((w, s))
            key = (use - 1, t, k)
            if key in last_writer:
                deps[(w, s)].add(last_writer[key])
            last_writer[key] = (w, s)
    succ = {v: [] for v in order}
    for v, ds in deps.items():
        for x in ds:
            if pos[x] >= pos[v]:
                raise ConfigurationError("launch schedule: dependency against the sweep order")
            succ[x].append(v)
    prio = {}
    for v in reversed(order):
        prio[v] = 1 + max((prio[x] for x in succ[v]), default=0)
    missing = {v: len(ds) for v, ds in deps.items()}
    ready = [v for v in order if missing[v] == 0]
    launches = []
    recent: list = []
    while ready:
        if resident > 0:
            hot = set(recent[-resident:])
            ready.sort(key=lambda v: (v[1] not in hot, -prio[v], pos[v]))
        else:
            ready.sort(key=lambda v: (-prio[v], pos[v]))
        pick, ready = ready[:cap], ready[cap:]
        pick.sort(key=lambda v: pos[v])
        launches.append(pick)
        if resident > 0:
            for v in pick:
                if v[1] in recent:
                    recent.remove(v[1])
                recent.append(v[1])
        for v in pick:
            for x in succ[v]:
                missing[x] -= 1
                if missing[x] == 0:
                    ready.append(x)
    if sum(len(l) for l in launches) != len(order):
        raise ConfigurationError("launch schedule: dependency cycle")
    return launches


class DevicePlan:
    """Static device tables for one (partition, operators, sweep plan).

    Built from the bit-exact host metadata: windows / owned regions /
    beta00 supports (partition.py), step groups (`_step_groups`,
    ddm.py:198-203), routing (`next_usable_sweep`, transfer.py:90-97) and
    psi geometry (transfer.py:100-155).
    """

    def __init__(self, partition, operators, cache, directions, nrhs_max: int,
                 schedule: str = "diagonal", pipelined: bool = False, shard=None,
                 pool_slots: int | None = None):
        """schedule "diagonal": one device sweep per sweep direction, visits
        grouped by anti-diagonal step (ddm.py:212-291).  schedule "additive":
        the additive overlapping DDM (ddm.py:294-349) on the same kernels --
        one device sweep per step, every subdomain visited, and a payload
        emitted at step s in direction d consumed at step s + |d|_1 (dropped
        silently past the last step, as the reference never reads it)."""
        from .partition import steps_per_sweep, sweep_step_of
        from .transfer import next_usable_sweep, transfer_geometry

        if schedule not in ("diagonal", "additive"):
            raise ConfigurationError(f"unknown DDM schedule {schedule!r}")
        self.schedule = schedule

        lib, ctx = context()
        dim = partition.dim
        subs = list(partition.subdomains())
        nsub = len(subs)
        lin = {idx: s for s, idx in enumerate(subs)}
        ops = [operators[idx] for idx in subs]
        # shard = (nranks, rank, owner[s]): this plan runs only its rank's
        # visits and factorizes only its rank's operators (sharded.py)
        self.shard = shard
        # pool_slots: out-of-core factors (FactorPool) -- the block LU of every
        # operator, `pool_slots` of them resident at a time, loaded launch by
        # launch (apply runs eagerly, launch by launch)
        self.pool = None
        if pool_slots is not None:
            if shard is not None or schedule != "diagonal":
                raise ConfigurationError("pooled factors: diagonal, unsharded plans only")
            self.pool = FactorPool(ops, pool_slots)
            facts = [_PoolRef(self.pool, i) for i in range(nsub)]
        elif shard is not None:
            nranks, rank, owner = shard
            owned = [s for s in range(nsub) if owner[s] == rank]
            ofacts = dict(zip(owned, cache.factorizations([ops[s] for s in owned])))
            facts = [ofacts.get(s) for s in range(nsub)]
        else:
            facts = cache.factorizations(ops)
        self.partition = partition
        self.dim = dim
        self.nsub = nsub
        total_steps = sum(partition.counts) - dim + 1
        self.nsweeps = len(directions) if schedule == "diagonal" else total_steps
        self.directions = tuple(directions) if schedule == "diagonal" else ()
        self.nrhs_max = nrhs_max
        self.nnodes = partition.grid.node_count()
        self._keep = [ops, facts]

        win_lo, win_shape, own_lo, own_shape, sup_lo, sup_shape = [], [], [], [], [], []
        beta_vals, beta_off = [], []
        off = 0
        for idx in subs:
            w = partition.window(idx)
            o = partition.owned_window(idx)
            sp = partition.beta00_window(idx)
            win_lo += _pad3(w.lo); win_shape += _pad3(w.shape, 1)
            own_lo += _pad3(o.lo); own_shape += _pad3(o.shape, 1)
            sup_lo += _pad3(sp.lo); sup_shape += _pad3(sp.shape, 1)
            ramps = partition.beta00_axis_values(idx)
            for a in range(3):
                beta_off.append(off)
                if a < dim:
                    beta_vals.append(np.asarray(ramps[a], dtype=np.float64))
                    off += ramps[a].size
        dirs = source_directions(dim)
        ndir = len(dirs)
        visit_sub, step_off = [], []
        if schedule == "additive":
            nsteps = 1
            order = [lin[i] for i in sorted(subs)]
            for _ in range(self.nsweeps):
                visit_sub += order
                step_off += [0, len(order)]
        else:
            nsteps = steps_per_sweep(partition.counts)
        for sd in self.directions:
            groups: dict = {}
            for idx in subs:
                groups.setdefault(sweep_step_of(idx, sd, partition.counts), []).append(idx)
            order = []
            offs = [0]
            for t in range(1, nsteps + 1):
                order += [lin[i] for i in sorted(groups.get(t, []))]
                offs.append(len(order))
            visit_sub += order
            step_off += offs
        geoms = {}
        band_lo, band_shape, ext_lo, ext_shape, xfac_off = [], [], [], [], []
        xfac_vals = []
        foff = 0
        for s, idx in enumerate(subs):
            for k, dvec in enumerate(dirs):
                g = transfer_geometry(partition, idx, dvec)
                geoms[(s, k)] = g
                if g is None:
                    band_lo += [0] * 3; band_shape += [0] * 3
                    ext_lo += [0] * 3; ext_shape += [0] * 3
                    xfac_off += [0] * 3
                    continue
                band_lo += _pad3(g.band.lo); band_shape += _pad3(g.band.shape, 1)
                ext_lo += _pad3(g.ext.lo); ext_shape += _pad3(g.ext.shape, 1)
                for a in range(3):
                    xfac_off.append(foff)
                    if a < dim:
                        xfac_vals.append(np.asarray(g.factors[a], dtype=np.float64))
                        foff += g.factors[a].size
        xfer_use = np.full((self.nsweeps, nsub, ndir), -1, dtype=np.int32)
        for w in range(self.nsweeps):
            for s in range(nsub):
                for k, dvec in enumerate(dirs):
                    if geoms[(s, k)] is None:
                        continue
                    if schedule == "additive":
                        use = w + 1 + sum(abs(c) for c in dvec)
                        xfer_use[w, s, k] = use if use <= self.nsweeps else -1
                        continue
                    use = next_usable_sweep(dvec, w + 1, self.directions)
                    xfer_use[w, s, k] = 0 if use is None else use
        self.xfer_use = xfer_use
        # ---- launch schedule: visits of several sweeps per launch as soon as
        # their sources are done (the dependency DAG of the sweep is shallower
        # than sweeps x steps); the cluster solve fits ~7 visits per wave
        self.launches = None
        if (pipelined or shard is not None or self.pool is not None) and schedule == "diagonal":
            order = []
            for w in range(self.nsweeps):
                b0 = w * (nsteps + 1)
                for t in range(nsteps):
                    for i in range(step_off[b0 + t], step_off[b0 + t + 1]):
                        order.append((w, visit_sub[w * nsub + i]))
            pc = partition.counts

            def sub_index(sv, d):
                idx = tuple(i + c for i, c in zip(subs[sv], d))
                return lin[idx]

            max_m = 0
            for idx in subs:
                shp = partition.window(idx).shape
                ax = int(np.argmax(shp))
                max_m = max(max_m, int(np.prod([n for a, n in enumerate(shp) if a != ax])))
            cap_env = os.environ.get("DS_LAUNCH_CAP")
            # cluster solve: 8 visits per launch (measured best on config 2:
            # 13.4 ms vs 14.2 at 7; 9-10 give the same as 8); staged 3D: unbounded
            cap = int(cap_env) if cap_env else (8 if max_m <= 160 else nsub * self.nsweeps)
            if self.pool is not None:
                # out of core: every miss is a factorization; factor-local order,
                # up to 8 visits per launch so a launch's misses are factored as one
                # batch (config 5: 415 factorizations per application at 0.75 s
                # each, 939 s for the GMRES solve, vs 2 visits per launch: 365
                # at 1.0 s, 1101 s -- K2b batches keep more GPCs busy)
                cap = min(int(cap_env) if cap_env else 8, self.pool.nslots)
            if not pipelined:  # sweep-ordered launches (one per (sweep, step))
                self.launches = []
                for w in range(self.nsweeps):
                    b0 = w * (nsteps + 1)
                    for t in range(nsteps):
                        self.launches.append([(w, visit_sub[w * nsub + i])
                                              for i in range(step_off[b0 + t], step_off[b0 + t + 1])])
            else:
                self.launches = launch_schedule(self.nsweeps, nsub, order, xfer_use, dirs, sub_index,
                                                None, max(1, cap),
                                                self.pool.nslots if self.pool is not None else 0)
            if shard is not None:  # same launch boundaries on every rank, own visits only
                self.launches = [[v for v in L if shard[2][v[1]] == shard[1]] for L in self.launches]
        self.pool_loads = None
        self.pool_seconds = 0.0  # host time spent factoring pool slots (pooled plans)
        if self.pool is not None:
            vslot, self.pool_loads, self.pool_misses = belady_slots(self.launches, self.pool.nslots)
            visit_slot = np.full(self.nsweeps * nsub, -1, np.int32)
            for (w, sv), c in vslot.items():
                visit_slot[w * nsub + sv] = c
        self.geoms = geoms
        self.subs = subs
        self.dirs = dirs
        self.nsteps = nsteps
        self.visit_sub = np.asarray(visit_sub, dtype=np.int32)
        self.step_off = np.asarray(step_off, dtype=np.int32)

        arrays = dict(
            win_lo=np.asarray(win_lo, np.int32), win_shape=np.asarray(win_shape, np.int32),
            own_lo=np.asarray(own_lo, np.int32), own_shape=np.asarray(own_shape, np.int32),
            sup_lo=np.asarray(sup_lo, np.int32), sup_shape=np.asarray(sup_shape, np.int32),
            beta00=np.concatenate(beta_vals), beta00_off=np.asarray(beta_off, np.int64),
            op_of_sub=np.arange(nsub, dtype=np.int32),
            fact_index=np.asarray([f.index if f is not None else 0 for f in facts], np.int32),
            visit_sub=self.visit_sub, step_off=self.step_off,
            directions=np.asarray([_pad3(dv) for dv in dirs], np.int32).ravel(),
            xfer_use=xfer_use.ravel(),
            band_lo=np.asarray(band_lo, np.int32), band_shape=np.asarray(band_shape, np.int32),
            ext_lo=np.asarray(ext_lo, np.int32), ext_shape=np.asarray(ext_shape, np.int32),
            xfac=np.concatenate(xfac_vals) if xfac_vals else np.zeros(1),
            xfac_off=np.asarray(xfac_off, np.int64),
        )
        dops = [device_operator(op) for op in ops]
        self._keep.append(dops)
        op_handles = (C.c_void_p * nsub)(*[d.handle.value for d in dops])
        fact_handles = (C.c_void_p * nsub)(*[f.fset.handle.value if f is not None else None
                                             for f in facts])
        desc = N.PlanDesc()
        desc.dim, desc.nsub, desc.nsweeps = dim, nsub, self.nsweeps
        desc.nsteps, desc.ndir, desc.nrhs_max = nsteps, ndir, nrhs_max
        for a in range(3):
            desc.grid_counts[a] = partition.grid.counts[a] if a < dim else 1
            desc.part_counts[a] = partition.counts[a] if a < dim else 1
        for name, arr in arrays.items():
            setattr(desc, name, arr.ctypes.data)
        desc.nops = nsub
        desc.ops = C.cast(op_handles, C.c_void_p)
        desc.fact_of_sub = C.cast(fact_handles, C.c_void_p)
        if shard is not None:
            owner_arr = np.asarray(shard[2], np.int32)
            arrays["owner"] = owner_arr  # keep alive
            desc.nranks, desc.rank, desc.owner = shard[0], shard[1], owner_arr.ctypes.data
        if self.pool is not None:
            arrays["visit_slot"] = visit_slot  # keep alive
            desc.visit_slot = visit_slot.ctypes.data
        if self.launches is not None:
            l_off = np.zeros(len(self.launches) + 1, np.int32)
            l_vis = []
            for i, L in enumerate(self.launches):
                l_off[i + 1] = l_off[i] + len(L)
                for (w, sv) in L:
                    l_vis += [w, sv]
            l_vis = np.asarray(l_vis, np.int32)
            arrays["launch_off"], arrays["launch_visits"] = l_off, l_vis  # keep alive
            desc.nlaunch = len(self.launches)
            desc.launch_off = l_off.ctypes.data
            desc.launch_visits = l_vis.ctypes.data
        out = C.c_void_p()
        N.check(lib.ds_plan_create(ctx, C.byref(desc), C.byref(out)), "ds_plan_create")
        self.handle = out
        self._finalizer = weakref.finalize(self, lib.ds_plan_destroy, out)
        # replay one captured CUDA graph per (buffers, nrhs): ~4 sweeps x
        # n_steps x 4 launches per application (DS_GRAPH=0 disables)
        if os.environ.get("DS_GRAPH", "1") != "0" and shard is None and self.pool is None:
            self.enable_graph(True)
        if self.pool is not None:
            sb, _, fb, _ = self.shard_info()
            self.set_peers([sb], [fb])  # one rank: launch-range execution

    @property
    def workspace_bytes(self) -> int:
        return N.load_library().ds_plan_workspace_bytes(self.handle)

    def enable_graph(self, enable: bool = True):
        lib, ctx = context()
        N.check(lib.ds_ddm_enable_graph(ctx, self.handle, int(bool(enable))))

    # ---- sharded plans (sharded.py)
    def shard_info(self):
        """(slot_base, slot_bytes, flag_base, flag_bytes) device memory peers write into."""
        lib = N.load_library()
        sb, fb = C.c_void_p(), C.c_void_p()
        sn, fn = C.c_int64(), C.c_int64()
        N.check(lib.ds_plan_shard_info(self.handle, C.byref(sb), C.byref(sn), C.byref(fb),
                                       C.byref(fn)), "ds_plan_shard_info")
        return sb.value, sn.value, fb.value, fn.value

    def set_peers(self, slot_bases, flag_bases):
        lib, ctx = context()
        n = len(slot_bases)
        sa = (C.c_void_p * n)(*slot_bases)
        fa = (C.c_void_p * n)(*flag_bases)
        N.check(lib.ds_plan_set_peers(ctx, self.handle, n, sa, fa), "ds_plan_set_peers")

    def slot(self, use_sweep: int, target: int, k: int, nrhs: int):
        """Band (lo, shape) and contents [*shape, nrhs] (CUDA tensor) of the
        payload slot for direction k queued for visit (use_sweep 1-based,
        target); None if no routing fills it (ds_plan_slot)."""
        lib, ctx = context()
        lo = (C.c_int32 * 3)()
        sh = (C.c_int32 * 3)()
        if lib.ds_plan_slot(ctx, self.handle, use_sweep, target, k, lo, sh, None, 0, nrhs) != 0:
            return None
        shape = tuple(sh[:self.dim])
        out = torch.empty(shape + (nrhs,), dtype=torch.complex128, device="cuda")
        N.check(lib.ds_plan_slot(ctx, self.handle, use_sweep, target, k, lo, sh, out.data_ptr(),
                                 out.numel(), nrhs), "ds_plan_slot")
        return tuple(lo[:self.dim]), shape, out

    def nlaunch(self) -> int:
        return int(N.load_library().ds_plan_nlaunch(self.handle))

    def apply_range(self, fmin, umin, nrhs: int, l0: int, l1: int, mode: int):
        lib, ctx = context()
        N.check(lib.ds_ddm_apply_range(ctx, self.handle, fmin.data_ptr(), umin.data_ptr(), nrhs,
                                       l0, l1, mode), "ds_ddm_apply_range")

    def last_launches(self) -> int:
        return N.load_library().ds_plan_last_launches(self.handle)

    def set_profiling(self, enable: bool = True):
        N.check(N.load_library().ds_plan_set_profiling(self.handle, int(bool(enable))))

    KERNEL_CLASSES = ("assemble", "block_solve", "accumulate", "transfer", "modal_recurrence")

    def kernel_times(self, reset: bool = True) -> dict:
        """{class: (total_ms, launches)} since the last reset (CUDA events);
        'block_solve' is K3 or the modal transforms (K3m-T)."""
        ms = (C.c_double * 5)()
        cnt = (C.c_int64 * 5)()
        N.check(N.load_library().ds_plan_kernel_times(self.handle, ms, cnt, int(reset)))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(self.KERNEL_CLASSES)}

    def apply_minor(self, fmin, umin, nrhs: int, partials=None):
        """One application on RHS-minor device buffers (no layout work)."""
        lib, ctx = context()
        if self.pool is not None:  # launch by launch, loading the slots each needs
            if partials is not None:
                raise ConfigurationError("pooled factors: no per-sweep partials")
            import time

            last = len(self.launches) - 1
            for l, loads in enumerate(self.pool_loads):
                t0 = time.perf_counter()
                self.pool.load_many(loads)  # synchronous: factors the slots' new owners
                self.pool_seconds += time.perf_counter() - t0
                self.apply_range(fmin, umin, nrhs, l, l + 1, (1 if l == 0 else 0) | (2 if l == last else 0))
            return
        N.check(lib.ds_ddm_apply(ctx, self.handle, fmin.data_ptr(), umin.data_ptr(), nrhs,
                                 0 if partials is None else partials.data_ptr()),
                "ds_ddm_apply")

    def _minor_buffers(self, R, device):
        """Persistent RHS-minor f/u buffers per batch size (stable pointers let
        the native side replay its captured CUDA graph)."""
        bufs = getattr(self, "_bufs", None)
        if bufs is None:
            bufs = self._bufs = {}
        if R not in bufs:
            fmin = torch.empty((self.nnodes, R), dtype=torch.complex128, device=device)
            bufs[R] = (fmin, torch.empty_like(fmin))
        return bufs[R]

    def apply(self, f, collect_partials: bool = False, out=None):
        """f: [R, N] complex128 CUDA tensor (RHS-outer) -> (u [R, N], partials);
        `out` (optional, contiguous [R, N]) receives u."""
        lib, ctx = context()
        R = f.shape[0]
        n = self.nnodes
        fmin, umin = self._minor_buffers(R, f.device)
        N.check(lib.ds_layout_to_minor(ctx, n, R, f.data_ptr(), fmin.data_ptr()))
        partials = None
        if collect_partials:
            partials = torch.empty((self.nsweeps, n, R), dtype=torch.complex128, device=f.device)
        self.apply_minor(fmin, umin, R, partials)
        u = out if out is not None else torch.empty((R, n), dtype=torch.complex128, device=f.device)
        N.check(lib.ds_layout_to_outer(ctx, n, R, umin.data_ptr(), u.data_ptr()))
        parts = None
        if partials is not None:
            parts = []
            for w in range(self.nsweeps):
                p = torch.empty((R, n), dtype=torch.complex128, device=f.device)
                N.check(lib.ds_layout_to_outer(ctx, n, R, partials[w].data_ptr(), p.data_ptr()))
                parts.append(p)
        return u, parts

    def apply_host(self, f_host, u_host):
        """One application from a pinned host tensor f_host [R, N] into the
        pinned host tensor u_host [R, N] (ds_ddm_apply_host: chunked uploads
        and downloads overlapped with the sweep); synchronous on return."""
        lib, ctx = context()
        R = f_host.shape[0]
        N.check(lib.ds_ddm_apply_host(ctx, self.handle, f_host.data_ptr(), u_host.data_ptr(), R),
                "ds_ddm_apply_host")
        torch.cuda.current_stream().synchronize()

    def counters(self, nrhs: int):
        lib, ctx = context()
        per = self.nsweeps * self.nsub * nrhs
        nonzero = np.zeros(nrhs, np.int32)
        discarded = np.zeros(nrhs, np.int32)
        vnz = np.zeros(per, np.int32)
        vcons = np.zeros(per, np.int32)
        vemit = np.zeros(per, np.int32)
        vcut = np.zeros(per, np.int32)
        P = N.P_i32
        N.check(lib.ds_ddm_counters(ctx, self.handle, nrhs, nonzero.ctypes.data_as(P),
                                    discarded.ctypes.data_as(P), vnz.ctypes.data_as(P),
                                    vcons.ctypes.data_as(P), vemit.ctypes.data_as(P),
                                    vcut.ctypes.data_as(P)), "ds_ddm_counters")
        shape = (self.nsweeps, self.nsub, nrhs)
        return dict(nonzero=nonzero, discarded=discarded, visit_nonzero=vnz.reshape(shape),
                    visit_consumed=vcons.reshape(shape), visit_emitted=vemit.reshape(shape),
                    visit_cut=vcut.reshape(shape))


class _PoolRef:
    """A subdomain's factors inside a FactorPool (DevicePlan's fact table)."""

    backend = "splu"
    device_backend = "block-lu"

    def __init__(self, pool, index):
        self.fset = pool
        self.index = index


class GroupedPlan:
    """RHS groups pipelined through the sweeps (the paper's Remark 2): the
    batch is split into `groups` contiguous RHS groups, each run by its own
    native plan on its own stream, so one group's latency-bound kernels
    (assembly, recurrences, transfers, small launches) overlap another
    group's transforms.  RHS are independent through the map and every
    group's arithmetic is the ungrouped arithmetic, so results are bitwise
    those of one plan over the whole batch (tools/split_probe.py; config 2
    +8%, config 3 DDM application +15% on a B200).  Counters / reports are
    concatenated along the RHS axis; other attributes are the first group's
    (identical static tables)."""

    def __init__(self, plans):
        self.plans = plans
        self.groups = len(plans)
        self._streams = [torch.cuda.Stream() for _ in plans]
        self._split = None

    def __getattr__(self, name):
        return getattr(self.plans[0], name)

    @property
    def nrhs_max(self):
        return sum(p.nrhs_max for p in self.plans)

    def _bounds(self, R):
        G = min(self.groups, R)
        return [(R * g // G, R * (g + 1) // G) for g in range(G)]

    def apply(self, f, collect_partials: bool = False):
        R = f.shape[0]
        if collect_partials or R < 2:
            return self.plans[0].apply(f, collect_partials)  # one group (nrhs_max covers it)
        bounds = self._bounds(R)
        main = torch.cuda.current_stream()
        u = torch.empty((R, f.shape[1]), dtype=torch.complex128, device=f.device)
        for (r0, r1), p, st in zip(bounds, self.plans, self._streams):
            st.wait_stream(main)
            with torch.cuda.stream(st):
                p.apply(f[r0:r1], out=u[r0:r1])  # each group writes its rows in place
        for st in self._streams[:len(bounds)]:
            main.wait_stream(st)
        context()  # leave the shared native context on the caller's stream
        self._split = bounds
        return u, None

    def apply_host(self, f_host, u_host):
        """Pinned host f [R, N] -> pinned host u: the groups sweep
        concurrently, one shared copy pipeline (ds_ddm_apply_host_groups)."""
        R = f_host.shape[0]
        G = min(self.groups, R)
        lib, ctx = context()
        arr = (C.c_void_p * G)(*[p.handle.value for p in self.plans[:G]])
        N.check(lib.ds_ddm_apply_host_groups(ctx, arr, G, f_host.data_ptr(), u_host.data_ptr(), R),
                "ds_ddm_apply_host_groups")
        torch.cuda.current_stream().synchronize()
        self._split = self._bounds(R)

    def counters(self, nrhs: int):
        bounds = self._split if self._split and self._split[-1][1] == nrhs else None
        if bounds is None:
            return self.plans[0].counters(nrhs)
        parts = [p.counters(r1 - r0) for (r0, r1), p in zip(bounds, self.plans)]
        return {k: np.concatenate([c[k] for c in parts], axis=-1) for k in parts[0]}

    def set_profiling(self, enable: bool = True):
        for p in self.plans:
            p.set_profiling(enable)

    def kernel_times(self, reset: bool = True) -> dict:
        out = {}
        for p in self.plans:
            for k, (ms, n) in p.kernel_times(reset).items():
                a, b = out.get(k, (0.0, 0))
                out[k] = (a + ms, b + n)
        return out

    def last_launches(self) -> int:
        return sum(p.last_launches() for p in self.plans)
