"""GPU factorization cache: the plugin point of the sweep engine.

Drop-in for `FactorizationCache` / `factorize` (diagsweep/subdomain.py:
139-179): `cache.get(op)` returns a factorization with `.solve(rhs)`,
`.backend`, `.factor_bytes`, keyed by `op.fingerprint` so operators with
identical coefficient bytes share one factorization (subdomain.py:153-171).

Backends (the reference's dispatch, subdomain.py:139-147: 'auto' picks
'separable' for tensor-structured kappa^2, else 'splu'):
* 'separable' -> the modal factorization (K2m/K3m, csrc/ds_modal.cu): the
  in-slab 1D tridiagonals are diagonalised (host LAPACK eig of n_a x n_a
  matrices, as the reference's own separable backend calls scipy.linalg.schur)
  and the device keeps the transforms and mode-wise pivots; solves are
  batched complex GEMMs on the FP64 tensor cores plus mode-wise recurrences.
* 'splu' / 'block-lu' -> the block-tridiagonal dense-block LU of K2
  (csrc/ds_factor.cu), for every operator kind (replaces SuperLU).
DS_FACTOR=block-lu in the environment makes 'auto' use the block LU for
every operator (A/B measurements).  `share_translates=True` (opt-in, off by default to keep the reference's
exact-fingerprint semantics) keys operators by their coefficients rounded to
12 significant digits, so windows that are translates of each other (equal
up to linspace round-off, ~1e-16) share one factorization.  This is what lets
config 4 (3D, 64 windows, 203 GB of dense factors) fit HBM: its 27
translation classes need ~76 GB (SURVEY §7 hard part 3); the perturbation of
a shared operator is ~1e-16 relative, far below the 1e-10 parity bar.
`method` keeps the reference's vocabulary and checks:
'separable' on a non-separable operator raises ConfigurationError
(subdomain.py:48-50), unknown methods raise ConfigurationError
(subdomain.py:146).  Factorizations of many operators are created in one
batched launch (`prepare`).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

from .errors import ConfigurationError

_METHODS = ("auto", "separable", "splu", "block-lu")


class GpuFactorization:
    def __init__(self, fset, index: int, op):
        self.backend = "separable" if getattr(fset, "modal", False) else "block-lu"
        self.fset = fset
        self.index = index
        self.window = op.window
        self.shape = op.window.shape
        self._op = op
        ba, nb, m, nbytes = fset.info(index)
        self.block_axis, self.n_blocks, self.block_size = ba, nb, m
        self.factor_bytes = nbytes

    def solve(self, rhs):
        """x = A^{-1} rhs; rhs `[*window]` or batched `[R, *window]`."""
        from . import _engine

        shape = tuple(rhs.shape)
        if shape != self.shape and shape[1:] != self.shape:
            raise ConfigurationError(
                f"rhs shape {shape} does not match window {self.shape}")
        return _engine.fact_solve(self.fset, self.index, self._op, rhs)


def _check_method(op, method: str):
    if method not in _METHODS:
        raise ConfigurationError(f"unknown factorization method {method!r}")
    if method == "separable" and not op.separable:
        raise ConfigurationError("operator kappa^2 is not tensor-structured")


def _resolve(op, method: str) -> bool:
    """True for the modal (separable) backend, False for the block LU."""
    _check_method(op, method)
    if method == "auto":
        if os.environ.get("DS_FACTOR", "") == "block-lu":
            return False
        return bool(op.separable)
    return method == "separable"


def factorize(op, method: str = "auto") -> GpuFactorization:
    """Factor one operator on the GPU (modal if separable, else block LU)."""
    from . import _engine

    return GpuFactorization(_engine.FactorSet([op], modal=_resolve(op, method)), 0, op)


def _coarse_key(op) -> str:
    """Coefficient key insensitive to last-bit round-off (translates share)."""
    import hashlib

    import numpy as np

    sha = hashlib.sha1()
    sha.update(repr((op.window.shape, op.kappa2_kind)).encode())

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

    for lo, hi in op.couplings:
        feed(lo)
        feed(hi)
    k2 = op.kappa2_array()
    feed(k2)
    return sha.hexdigest()


@dataclass
class FactorizationCache:
    method: str = "auto"
    share_translates: bool = False
    _store: dict = field(default_factory=dict)
    hits: int = 0
    misses: int = 0
    _plans: dict = field(default_factory=dict, repr=False)

    def prepare(self, ops) -> None:
        """Factor every not-yet-cached distinct operator in one batched launch."""
        from . import _engine

        todo = {}
        for op in ops:
            _check_method(op, self.method)
            key = self.key(op)
            if key not in self._store and key not in todo:
                todo[key] = op
        if not todo:
            return
        for modal in (True, False):
            group = [(k, op) for k, op in todo.items() if _resolve(op, self.method) == modal]
            if not group:
                continue
            fset = _engine.FactorSet([op for _, op in group], modal=modal)
            for i, (key, op) in enumerate(group):
                self._store[key] = GpuFactorization(fset, i, op)

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
