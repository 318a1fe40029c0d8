"""GPU factorization cache: the plugin point of the sweep engine.

Drop-in for `FactorizationCache` / `factorize` (diagsweep/subdomain.py:
139-179): `cache.get(op)` returns a factorization with `.solve(rhs)`,
`.backend`, `.factor_bytes`, keyed by `op.fingerprint` so operators with
identical coefficient bytes share one factorization (subdomain.py:153-171).
`op` may be this package's `DiscreteOperator` or the reference's own: only
the reference's public operator surface is read (`window`, `grid`,
`axis_coefficients(a)`, `kappa2_kind`, `kappa2`, `fingerprint`,
pml.py:75-113).

Backends keep the reference's names and dispatch (subdomain.py:139-147:
'auto' picks 'separable' for tensor-structured kappa^2, else 'splu'):
* backend 'separable' -> the modal factorization (K2m/K3m, csrc/ds_modal.cu):
  the in-slab 1D tridiagonals are diagonalised (host LAPACK eig of n_a x n_a
  matrices, as the reference's own separable backend calls
  scipy.linalg.schur) and the device keeps the transforms and mode-wise
  pivots; solves are batched complex GEMMs on the FP64 tensor cores plus
  mode-wise recurrences.  Guarded: when an eigenbasis is ill-conditioned
  (cond(V) > `modal_cond_max`, default 1e6) or the decomposition residuals
  are large (`_engine.modal_guard`), that operator falls back to the block
  LU, and `.fallback` says why.
* backend 'splu' -> the block-tridiagonal dense-block LU of K2
  (csrc/ds_factor.cu), the replacement of SuperLU for every operator kind;
  `.device_backend` is 'block-lu'.  `method='block-lu'` is accepted as an
  alias of 'splu' for separable operators too (A/B measurements).
`share_translates=True` (opt-in, off by default to keep the reference's
exact-fingerprint semantics) keys operators by their coefficients rounded to
12 significant digits, so windows that are translates of each other (equal
up to linspace round-off, ~1e-16) share one factorization (block-LU runs of
constant 3D media: config 4's 27 translation classes need ~76 GB of dense
factors instead of 203 GB).
`method` keeps the reference's vocabulary and checks: 'separable' on a
non-separable operator raises ConfigurationError (subdomain.py:48-50),
unknown methods raise ConfigurationError (subdomain.py:146).
Factorizations of many operators are created in one batched launch
(`prepare`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError

_METHODS = ("auto", "separable", "splu", "block-lu")


class GpuFactorization:
    """One operator's factors inside a batched device factor set."""

    def __init__(self, fset, index: int, op, fallback: str = ""):
        self.device_backend = "modal" if getattr(fset, "modal", False) else "block-lu"
        # the reference's backend names (subdomain.py:47, :112)
        self.backend = "separable" if self.device_backend == "modal" else "splu"
        self.fallback = fallback
        self.fset = fset
        self.index = index
        self.window = op.window
        self.shape = tuple(op.window.shape)
        self._dop = fset._dops[index]
        ba, nb, m, nbytes = fset.info(index)
        self.block_axis, self.n_blocks, self.block_size = ba, nb, m
        self.factor_bytes = nbytes
        # SparseLuFactorization's counters (subdomain.py:117-127): nonzeros
        # of the window matrix (5/7-point stencil) and stored factor entries
        W = int(np.prod(self.shape))
        self.matrix_nnz = W + 2 * sum(W // n * (n - 1) for n in self.shape)
        self.factor_nnz = nbytes // 16

    def solve(self, rhs):
        """x = A^{-1} rhs; rhs `[*window]` or batched `[R, *window]`."""
        from . import _engine

        shape = tuple(rhs.shape)
        if shape != self.shape and shape[1:] != self.shape:
            raise ConfigurationError(
                f"rhs shape {shape} does not match window {self.shape}")
        return _engine.fact_solve(self.fset, self.index, self.shape, rhs)


def _check_method(op, method: str):
    if method not in _METHODS:
        raise ConfigurationError(f"unknown factorization method {method!r}")
    if method == "separable" and not op.separable:
        raise ConfigurationError("operator kappa^2 is not tensor-structured")


def _wants_modal(op, method: str) -> bool:
    """The reference's dispatch: True for the separable backend."""
    _check_method(op, method)
    if method == "auto":
        return bool(op.separable)
    return method == "separable"


def factorize(op, method: str = "auto", modal_cond_max: float | None = None) -> GpuFactorization:
    """Factor one operator on the GPU (modal if separable and well
    conditioned, else block LU)."""
    cache = FactorizationCache(method=method, modal_cond_max=modal_cond_max)
    return cache.get(op)


def _coarse_key(op) -> str:
    """Coefficient key insensitive to last-bit round-off (translates share)."""
    import hashlib

    from ._engine import op_couplings, op_kappa2

    sha = hashlib.sha1()
    sha.update(repr((tuple(op.window.shape), op.kappa2_kind)).encode())

    def feed(a):
        a = np.asarray(a)
        if np.iscomplexobj(a):
            feed(a.real)
            feed(a.imag)
            return
        a = a.astype(np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            mag = np.where(a == 0, 0.0, np.floor(np.log10(np.abs(a))))
        q = np.where(a == 0, 0.0, np.round(a / 10.0 ** (mag - 11)))
        sha.update(q.astype(np.int64).tobytes())
        sha.update(mag.astype(np.int64).tobytes())

    for lo, hi in op_couplings(op):
        feed(lo)
        feed(hi)
    feed(op_kappa2(op)[2])
    return sha.hexdigest()


@dataclass
class FactorizationCache:
    method: str = "auto"
    share_translates: bool = False
    modal_cond_max: float | None = None  # None: _engine.MODAL_COND_MAX
    # out-of-core factors: when the block-LU factors of a plan's distinct
    # operators exceed `device_budget` bytes (None: free device memory minus
    # `pool_reserve`), the sweep plan keeps them in a FactorPool of as many
    # slots as fit and factors them launch by launch (config 5)
    device_budget: int | None = None
    pool_reserve: int = 32 << 30
    _store: dict = field(default_factory=dict)
    hits: int = 0
    misses: int = 0
    _plans: dict = field(default_factory=dict, repr=False)

    def prepare(self, ops) -> None:
        """Factor every not-yet-cached distinct operator in one batched launch
        per backend."""
        from . import _engine

        todo = {}
        for op in ops:
            _check_method(op, self.method)
            key = self.key(op)
            if key not in self._store and key not in todo:
                todo[key] = op
        if not todo:
            return
        cond_max = _engine.MODAL_COND_MAX if self.modal_cond_max is None else self.modal_cond_max
        modal, blocked = [], []
        for key, op in todo.items():
            if not _wants_modal(op, self.method):
                blocked.append((key, op, ""))
                continue
            ok, why, dec = _engine.modal_guard(op, cond_max)
            if ok:
                modal.append((key, op, dec))
            else:  # ill-conditioned eigenbasis: the block LU keeps 1e-10
                blocked.append((key, op, "modal factorization rejected: " + why))
        if modal:
            fset = _engine.FactorSet([op for _, op, _ in modal], modal=True,
                                     decomps=[dec for _, _, dec in modal])
            for i, (key, op, _) in enumerate(modal):
                self._store[key] = GpuFactorization(fset, i, op)
        if blocked:
            fset = _engine.FactorSet([op for _, op, _ in blocked], modal=False)
            for i, (key, op, why) in enumerate(blocked):
                self._store[key] = GpuFactorization(fset, i, op, fallback=why)

    def pool_slots(self, ops):
        """Slots of an out-of-core factor pool for these operators, or None
        when their factors fit (or some operator takes the modal backend)."""
        from . import _engine

        if any(_wants_modal(op, self.method) for op in ops):
            return None
        if all(self.key(op) in self._store for op in ops):
            return None
        shapes = {self.key(op): tuple(op.window.shape) for op in ops}
        need = sum(_engine.block_lu_bytes(sh) for sh in shapes.values())
        budget = self.device_budget
        if budget is None:
            import torch

            free, _ = torch.cuda.mem_get_info()
            budget = free - self.pool_reserve
        if need <= budget:
            return None
        per = max(_engine.block_lu_bytes(sh) for sh in shapes.values())
        nslots = int(budget // per)
        if nslots < 1:
            raise ConfigurationError(
                f"factor pool: one window's factors ({per / 1e9:.1f} GB) exceed the device budget")
        return nslots

    def key(self, op) -> str:
        return _coarse_key(op) if self.share_translates else op.fingerprint

    def get(self, op) -> GpuFactorization:
        key = self.key(op)
        fact = self._store.get(key)
        if fact is None:
            self.prepare([op])
            fact = self._store[key]
            self.misses += 1
        else:
            self.hits += 1
        return fact

    def factorizations(self, ops) -> list:
        """Factorizations for a list of operators (batched, counts like get)."""
        missing = {self.key(op) for op in ops if self.key(op) not in self._store}
        self.prepare(ops)
        out = []
        seen = set()
        for op in ops:
            key = self.key(op)
            if key in missing and key not in seen:
                self.misses += 1
                seen.add(key)
            else:
                self.hits += 1
            out.append(self._store[key])
        return out

    @property
    def count(self) -> int:
        return len(self._store)

    @property
    def total_bytes(self) -> int:
        return sum(f.factor_bytes for f in self._store.values())


def solve(fact, rhs):
    return fact.solve(rhs)
