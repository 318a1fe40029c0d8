"""The reference's plugin seam: `FactorizationCache.get(op)`
and the sweep accept the reference's own `DiscreteOperator`, reading only its
public surface (`window`, `grid`, `axis_coefficients(a)`, `kappa2_kind`,
`kappa2`, `fingerprint`; diagsweep/pml.py:75-113, subdomain.py:153-171,
ddm.py:216,259).  `ForeignOperator` below is a stand-in with exactly that
surface -- an unhashable dataclass like the reference's, without this
package's `couplings` / `kappa2_array` / `_device` extensions."""

import hashlib
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import pytest

from oracle import ds_oracle as O
from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve
from paper_2002_05327_b200 import _engine
from paper_2002_05327_b200.subdomain import _coarse_key


@dataclass
class ForeignOperator:
    grid: object
    window: object
    box: object
    alpha_nodes: list
    alpha_faces: list
    kappa2_kind: str
    kappa2: object

    @property
    def dim(self):
        return self.grid.dim

    @property
    def separable(self):
        return self.kappa2_kind != "full"

    def axis_coefficients(self, axis):
        h = self.grid.spacing[axis]
        node, face = self.alpha_nodes[axis], self.alpha_faces[axis]
        return 1.0 / (node * face[:-1] * h * h), 1.0 / (node * face[1:] * h * h)

    @cached_property
    def fingerprint(self):
        d = hashlib.sha1()
        d.update(repr((self.window.shape, self.kappa2_kind, self.grid.spacing)).encode())
        for arr in (*self.alpha_nodes, *self.alpha_faces):
            d.update(arr.tobytes())
        if self.kappa2_kind == "const":
            d.update(repr(self.kappa2).encode())
        elif self.kappa2_kind == "axis":
            d.update(repr(self.kappa2[0]).encode())
            d.update(self.kappa2[1].tobytes())
        else:
            d.update(self.kappa2.tobytes())
        return d.hexdigest()


def foreign(op):
    return ForeignOperator(op.grid, op.window, op.box, op.alpha_nodes, op.alpha_faces,
                           op.kappa2_kind, op.kappa2)


@pytest.fixture(scope="module")
def cfg1():
    s = configs.spec(1)
    return s, configs.build(s)


def test_foreign_operator_surface_matches_ours(cfg1):
    """Host side (no GPU): couplings, kappa^2 table, fingerprint and the
    translation key read through the public surface equal our operator's."""
    s, b = cfg1
    with pytest.raises(TypeError):
        hash(foreign(b["gop"]))  # unhashable, like the reference dataclass
    for idx in [(1, 1), (2, 3), (4, 4)]:
        op = b["ops"][idx]
        fo = foreign(op)
        assert not hasattr(fo, "couplings") and not hasattr(fo, "_device")
        for (a_lo, a_hi), (b_lo, b_hi) in zip(_engine.op_couplings(fo), op.couplings):
            assert np.array_equal(a_lo, b_lo) and np.array_equal(a_hi, b_hi)
        k_f, k_o = _engine.op_kappa2(fo), _engine.op_kappa2(op)
        assert k_f[:2] == k_o[:2] and np.array_equal(k_f[2], k_o[2])
        assert fo.fingerprint == op.fingerprint
        assert _coarse_key(fo) == _coarse_key(op)
        assert np.array_equal(_engine.axis_tridiagonal(fo, 0), _engine.axis_tridiagonal(op, 0))


def test_to_sparse_and_tridiag_dense_match_the_operator(cfg1):
    """pml.py:104-113,161-173 restated: the sparse window matrix times v is
    the oracle's stencil action; T_axis is the kappa-free 1D operator."""
    s, b = cfg1
    prob = O.Problem(**configs.oracle_problem(s, b))
    idx = (2, 3)
    op = b["ops"][idx]
    oop = prob.operators()[idx]
    A = op.to_sparse()
    assert A.shape == (op.window.size, op.window.size)
    rng = np.random.default_rng(2)
    v = rng.standard_normal(op.window.shape) + 1j * rng.standard_normal(op.window.shape)
    want = oop.apply(v)
    assert np.linalg.norm(A @ v.ravel() - want.ravel()) <= 1e-13 * np.linalg.norm(want)
    for a in range(2):
        T = op.tridiag_dense(a)
        assert np.array_equal(T, oop.tridiag(a))


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["auto", "splu"])
def test_gpu_cache_and_sweep_take_the_reference_operator(cuda, cfg1, method):
    """`cache.get(foreign_op).solve(rhs)` and `diagonal_sweep_solve` over a
    dict of foreign operators: results equal to our operators' bitwise and to
    the oracle within 1e-10; backend names are the reference's."""
    s, b = cfg1
    prob = O.Problem(**configs.oracle_problem(s, b))
    oops = prob.operators()
    cache = FactorizationCache(method=method)
    rng = np.random.default_rng(8)
    idx = (2, 2)
    fo = foreign(b["ops"][idx])
    fact = cache.get(fo)
    assert fact.backend == ("separable" if method == "auto" else "splu")
    assert cache.get(fo) is fact and cache.hits == 1 and cache.misses == 1
    rhs = rng.standard_normal(fo.window.shape) + 1j * rng.standard_normal(fo.window.shape)
    x = fact.solve(rhs)
    ref = O.factorize(oops[idx]).solve(rhs)
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)
    assert fact.matrix_nnz == oops[idx].to_sparse().nnz
    fops = {i: foreign(op) for i, op in b["ops"].items()}
    f = configs.sources(s, b["grid"])[0]
    u_f, rep_f = diagonal_sweep_solve(f, b["partition"], fops, FactorizationCache(method=method),
                                      warn_collar=False)
    u_o, rep_o = diagonal_sweep_solve(f, b["partition"], b["ops"], FactorizationCache(method=method),
                                      warn_collar=False)
    assert np.array_equal(u_f.values, u_o.values)
    want, orep = O.ddm_apply(prob, oops, O.Cache(), f)
    assert np.linalg.norm(u_f.values - want) <= 1e-10 * np.linalg.norm(want)
    assert rep_f.nonzero_solves == orep["nonzero_solves"]
