"""Host logic of the modal factorization (CPU, no GPU): the per-axis 1D
tridiagonals and their eigen-decompositions, and a NumPy restatement of the
modal solve (in-slab transforms + mode-wise tridiagonal LU without pivoting,
the algorithm of csrc/ds_modal.cu) against the oracle's Schur/Sylvester
separable solver (subdomain.py:43-96).  Test infrastructure only."""

import numpy as np
import pytest

from oracle import ds_oracle as O
from paper_2002_05327_b200 import configs
from paper_2002_05327_b200._engine import axis_tridiagonal, block_axis_of, modal_decomposition


@pytest.fixture(scope="module")
def cfg1():
    s = configs.spec(1)
    b = configs.build(s)
    prob = O.Problem(**configs.oracle_problem(s, b))
    return b, prob.operators()


def kron_apply(op, x):
    """L x with L = sum_a T_a (Kronecker sum) + kappa^2 (const)."""
    out = np.zeros_like(x)
    for a in range(op.dim):
        T = axis_tridiagonal(op, a)
        out += np.moveaxis(np.tensordot(T, np.moveaxis(x, a, 0), axes=(1, 0)), 0, a)
    if op.kappa2_kind == "const":
        out += float(op.kappa2) * x
    return out


def modal_solve(op, g):
    """NumPy restatement of K3m: W transforms, mode-wise LU, V transforms."""
    ba, axes = modal_decomposition(op)
    others = [a for a in range(op.dim) if a != ba]
    x = g.astype(np.complex128)
    for a, (V, W, lam, _q) in zip(others, axes):
        x = np.moveaxis(np.tensordot(W, np.moveaxis(x, a, 0), axes=(1, 0)), 0, a)
    lo, hi = op.couplings[ba]
    d = -(lo + hi) + (float(op.kappa2) if op.kappa2_kind == "const" else 0.0)
    mu = 0
    for a, (V, W, lam, _q) in zip(others, axes):
        sh = [1] * op.dim
        sh[a] = -1
        mu = mu + lam.reshape(sh)
    xm = np.moveaxis(x, ba, 0)
    mum = np.moveaxis(np.broadcast_to(mu, x.shape), ba, 0)[0]
    n = xm.shape[0]
    y = np.empty_like(xm)
    piv = d[0] + mum
    y[0] = xm[0]
    pivs = [piv]
    for k in range(1, n):
        mul = lo[k] / pivs[-1]
        pivs.append(d[k] + mum - mul * hi[k - 1])
        y[k] = xm[k] - mul * y[k - 1]
    y[n - 1] = y[n - 1] / pivs[n - 1]
    for k in range(n - 2, -1, -1):
        y[k] = (y[k] - hi[k] * y[k + 1]) / pivs[k]
    x = np.moveaxis(y, 0, ba)
    for a, (V, W, lam, _q) in zip(others, axes):
        x = np.moveaxis(np.tensordot(V, np.moveaxis(x, a, 0), axes=(1, 0)), 0, a)
    return x


def test_axis_tridiagonals_reproduce_the_operator(cfg1):
    b, oops = cfg1
    rng = np.random.default_rng(3)
    for idx in list(b["ops"])[:3]:
        op = b["ops"][idx]
        v = rng.standard_normal(op.window.shape) + 1j * rng.standard_normal(op.window.shape)
        ref = oops[idx].apply(v)
        assert np.linalg.norm(kron_apply(op, v) - ref) <= 1e-13 * np.linalg.norm(ref)


def test_modal_decomposition(cfg1):
    b, _ = cfg1
    for idx in list(b["ops"])[:3]:
        op = b["ops"][idx]
        ba, axes = modal_decomposition(op)
        assert ba == block_axis_of(op.window.shape)
        assert len(axes) == op.dim - 1
        others = [a for a in range(op.dim) if a != ba]
        for a, (V, W, lam, _q) in zip(others, axes):
            T = axis_tridiagonal(op, a)
            assert np.linalg.norm(V @ np.diag(lam) @ W - T) <= 1e-10 * np.linalg.norm(T)
            assert np.linalg.norm(W @ V - np.eye(len(lam))) <= 1e-10


def test_modal_solve_matches_separable_oracle(cfg1):
    b, oops = cfg1
    rng = np.random.default_rng(9)
    for idx in list(b["ops"])[:4]:
        op = b["ops"][idx]
        g = rng.standard_normal(op.window.shape) + 1j * rng.standard_normal(op.window.shape)
        ref = O.factorize(oops[idx]).solve(g)
        x = modal_solve(op, g)
        assert np.linalg.norm(x - ref) <= 1e-11 * np.linalg.norm(ref)


def test_modal_guard_quality_numbers(cfg1):
    """The guard's numbers on config 1 (cond(V) ~ 3e3): accepted; a tiny
    cond limit rejects with the reason."""
    from paper_2002_05327_b200._engine import modal_guard

    b, _ = cfg1
    op = b["ops"][(2, 2)]
    ok, why, (ba, axes) = modal_guard(op)
    assert ok and why == ""
    cond, res, inv_err = axes[0][3]
    assert 1.0 < cond < 1e5 and res < 1e-13 and inv_err < 1e-10
    ok, why, _ = modal_guard(op, cond_max=10.0)
    assert not ok and "cond(V)" in why


def test_modal_guard_rejects_defective_axis():
    """A defective 1D matrix (Jordan block: eigenvectors numerically
    parallel) fails the guard instead of silently losing digits."""
    from paper_2002_05327_b200._engine import _axis_eig

    n = 12
    T = np.eye(n, dtype=np.complex128) * (2 + 1j) + np.diag(np.ones(n - 1), 1)
    V, W, lam, (cond, res, inv_err) = _axis_eig(T)
    assert not (cond <= 1e6 and inv_err <= 1e-9)
