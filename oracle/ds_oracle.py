"""CPU ORACLE — test infrastructure only, never part of the product path.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
leg and `--impl reference`) may import this module.  It restates, in plain
NumPy/SciPy, the reference algorithm of the hot path
(`/root/reference/pkg/src/diagsweep`, pure Python; citations below are
file:line in that package).  The dense/sparse kernels it calls are the same
third-party routines the reference calls (NumPy `@`/`einsum`, LAPACK zgees
via `scipy.linalg.schur`, LAPACK ztrsyl, SuperLU via `splu`; versions are
unpinned in `pkg/pyproject.toml:10-13` — numpy>=1.24, scipy>=1.10 — the
container has NumPy 2.3.5 / SciPy 1.18.1).

Parity is pinned: `tests/golden/make_golden.py` imported the reference
itself in the build container and stored its outputs under `tests/golden/`;
`tests/test_oracle_golden.py` checks this restatement against them
(metadata and coefficients bit-exact, solutions to round-off).

Functions are self-contained (no import of the product package) so that the
oracle is an independent check of the product's host metadata as well.
"""

from __future__ import annotations

import itertools
import math
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy.linalg import get_lapack_funcs, schur

# ------------------------------------------------------------------ grid
# grid.py:20-43: nodes a + i*h, h = (b-a)/(n-1), np.linspace


class Problem:
    """Everything the hot path needs, built from raw parameters."""

    def __init__(self, extents, counts, part_counts, d, pml, sigma_max, exponent, omega,
                 velocity, collar=None):
        self.extents = tuple((float(a), float(b)) for a, b in extents)
        self.counts = tuple(int(n) for n in counts)
        self.dim = len(self.counts)
        self.spacing = tuple((b - a) / (n - 1) for (a, b), n in zip(self.extents, self.counts))
        self.part_counts = tuple(part_counts)
        self.d = int(d)
        self.pml = int(pml)
        self.collar = self.pml if collar is None else int(collar)
        self.sigma_max = float(sigma_max)
        self.exponent = int(exponent)
        self.omega = float(omega)
        self.velocity = velocity  # ("const", c) | ("layered", depths, speeds) | ("raster", extents, samples)
        # partition.py:169-206
        self.breaks = []
        for a, n_sub in enumerate(self.part_counts):
            cells = self.counts[a] - 1 - 2 * self.collar
            assert cells >= n_sub and cells % n_sub == 0
            per = cells // n_sub
            self.breaks.append(tuple(self.collar + i * per for i in range(n_sub + 1)))
        self.breaks = tuple(self.breaks)
        self.subdomains = list(itertools.product(*(range(1, n + 1) for n in self.part_counts)))

    def coords(self, a):
        return np.linspace(self.extents[a][0], self.extents[a][1], self.counts[a])

    # partition.py:77-104 -------------------------------------------------
    def box(self, idx):
        return (tuple(self.breaks[a][i - 1] for a, i in enumerate(idx)),
                tuple(self.breaks[a][i] for a, i in enumerate(idx)))

    def window(self, idx):
        reach = self.d + self.pml
        lo = tuple(self.breaks[a][i - 1] - reach if i > 1 else 0 for a, i in enumerate(idx))
        hi = tuple(self.breaks[a][i] + reach if i < self.part_counts[a] else self.counts[a] - 1
                   for a, i in enumerate(idx))
        return lo, hi

    def owned(self, idx):
        """restrict_source's owned window incl. the collar (ddm.py:185-194)."""
        lo, hi = [], []
        for a, i in enumerate(idx):
            bk = self.breaks[a]
            s = bk[i - 1] + 1 if i > 1 else bk[0]
            e = bk[i]
            lo.append(s if i > 1 else 0)
            hi.append(e if i < self.part_counts[a] else self.counts[a] - 1)
        return tuple(lo), tuple(hi)

    def interior(self):
        return tuple(b[0] for b in self.breaks), tuple(b[-1] for b in self.breaks)

    def interior_box(self):
        lo, hi = self.interior()
        return tuple((self.coords(a)[lo[a]], self.coords(a)[hi[a]]) for a in range(self.dim))

    # partition.py:26-32, :119-150 -----------------------------------------
    @staticmethod
    def beta_hat(t):
        t = np.clip(np.asarray(t, dtype=float), 0.0, 1.0)
        return 1.0 - t**3 * (10.0 - 15.0 * t + 6.0 * t * t)

    def beta_1d_nodes(self, axis, sign, i, nodes):
        nodes = np.asarray(nodes)
        bk = self.breaks[axis]
        if sign == -1 and i != 1:
            return self.beta_hat((bk[i - 1] - nodes) / self.d)
        if sign == 1 and i != self.part_counts[axis]:
            return self.beta_hat((nodes - bk[i]) / self.d)
        return np.ones(nodes.shape)

    def beta00_support(self, idx):
        wlo, whi = self.window(idx)
        lo = tuple(self.breaks[a][i - 1] - self.d if i > 1 else wlo[a] for a, i in enumerate(idx))
        hi = tuple(self.breaks[a][i] + self.d if i < self.part_counts[a] else whi[a]
                   for a, i in enumerate(idx))
        vals = np.ones(tuple(h - l + 1 for l, h in zip(lo, hi)))
        for a, i in enumerate(idx):
            nodes = np.arange(lo[a], hi[a] + 1)
            shape = [1] * self.dim
            shape[a] = -1
            vals = vals * (self.beta_1d_nodes(a, -1, i, nodes)
                           * self.beta_1d_nodes(a, 1, i, nodes)).reshape(shape)
        return (lo, hi), vals

    # media.py:60-101 (raster), :32-58 (layered) ---------------------------
    def speed(self, mesh_coords):
        kind = self.velocity[0]
        if kind == "const":
            return np.full(mesh_coords.shape[:-1], self.velocity[1])
        if kind == "layered":
            depths, speeds = self.velocity[1], self.velocity[2]
            k = np.searchsorted(np.asarray(depths), mesh_coords[..., -1], side="right")
            return np.asarray(speeds)[k]
        _, extents, samples = self.velocity
        counts = samples.shape
        base, frac = [], []
        for a, ((lo, hi), n) in enumerate(zip(extents, counts)):
            t = np.clip((mesh_coords[..., a] - lo) / (hi - lo) * (n - 1), 0.0, n - 1.0)
            i0 = np.minimum(t.astype(np.int64), n - 2) if n > 1 else np.zeros_like(t, np.int64)
            base.append(i0)
            frac.append(t - i0)
        out = np.zeros(mesh_coords.shape[:-1])
        for corner in range(1 << len(counts)):
            w = np.ones(mesh_coords.shape[:-1])
            ix = []
            for a in range(len(counts)):
                up = corner >> a & 1
                if up and counts[a] > 1:
                    ix.append(base[a] + 1)
                    w = w * frac[a]
                else:
                    ix.append(base[a])
                    if counts[a] > 1:
                        w = w * (1.0 - frac[a])
                    elif up:
                        w = w * 0.0
            out += w * samples[tuple(ix)].astype(np.float64)
        return out

    # pml.py:216-266 -------------------------------------------------------
    def operator(self, win, box, clamp_box=None):
        wlo, whi = win
        blo, bhi = box
        if clamp_box is None:
            clamp_box = tuple((self.coords(a)[blo[a]], self.coords(a)[bhi[a]])
                              for a in range(self.dim))
        an, af = [], []
        for a in range(self.dim):
            h = self.spacing[a]
            x = self.coords(a)
            s_lo = blo[a] - wlo[a] - self.pml
            s_hi = whi[a] - bhi[a] - self.pml
            assert s_lo >= 0 and s_hi >= 0
            if s_lo > 0:
                s_lo += 1
            if s_hi > 0:
                s_hi += 1
            nodes = x[wlo[a]: whi[a] + 1]
            faces = np.concatenate([nodes - h / 2, [nodes[-1] + h / 2]])

            def ramp(t, shift):
                s = (np.asarray(t, dtype=float) - shift * h) / (self.pml * h)
                return self.sigma_max * np.clip(s, 0.0, 1.0) ** self.exponent

            def sig(t):
                return ramp(x[blo[a]] - t, s_lo) + ramp(t - x[bhi[a]], s_hi)

            an.append(1.0 + 1j * sig(nodes))
            af.append(1.0 + 1j * sig(faces))
        cs = [np.clip(self.coords(a)[wlo[a]: whi[a] + 1], clamp_box[a][0], clamp_box[a][1])
              for a in range(self.dim)]
        kind = self.velocity[0]
        if kind == "const":
            k2 = ("const", (self.omega / self.velocity[1]) ** 2)
        elif kind == "layered":
            ax = self.dim - 1
            k = np.searchsorted(np.asarray(self.velocity[1]), cs[ax], side="right")
            k2 = ("axis", (ax, (self.omega / np.asarray(self.velocity[2])[k]) ** 2))
        else:
            mesh = np.stack(np.meshgrid(*cs, indexing="ij"), axis=-1)
            k2 = ("full", (self.omega / self.speed(mesh)) ** 2)
        return Op(self, win, an, af, k2)

    def operators(self):
        clamp = self.interior_box()
        return {idx: self.operator(self.window(idx), self.box(idx), clamp)
                for idx in self.subdomains}

    def global_operator(self):
        full = (tuple(0 for _ in self.counts), tuple(n - 1 for n in self.counts))
        return self.operator(full, self.interior(), self.interior_box())


class Op:
    """DiscreteOperator restated (pml.py:75-188)."""

    def __init__(self, prob, win, alpha_nodes, alpha_faces, kappa2):
        self.prob = prob
        self.lo, self.hi = win
        self.shape = tuple(h - l + 1 for l, h in zip(self.lo, self.hi))
        self.dim = len(self.shape)
        self.alpha_nodes = alpha_nodes
        self.alpha_faces = alpha_faces
        self.kappa2_kind, self.kappa2 = kappa2

    def couplings(self, a):  # pml.py:95-102
        h = self.prob.spacing[a]
        node, face = self.alpha_nodes[a], self.alpha_faces[a]
        return 1.0 / (node * face[:-1] * h * h), 1.0 / (node * face[1:] * h * h)

    def k2_on(self, rlo, rshape):
        sl = tuple(slice(l - w, l - w + n) for l, w, n in zip(rlo, self.lo, rshape))
        if self.kappa2_kind == "const":
            return self.kappa2
        if self.kappa2_kind == "axis":
            ax, vals = self.kappa2
            shape = [1] * self.dim
            shape[ax] = -1
            return vals[sl[ax]].reshape(shape)
        return self.kappa2[sl]

    def apply(self, v, rlo=None):  # pml.py:135-159
        if rlo is None:
            rlo = self.lo
        rshape = v.shape
        out = self.k2_on(rlo, rshape) * v
        for a in range(self.dim):
            c_lo, c_hi = self.couplings(a)
            s = rlo[a] - self.lo[a]
            c_lo = c_lo[s: s + rshape[a]]
            c_hi = c_hi[s: s + rshape[a]]
            shape = [1] * self.dim
            shape[a] = -1
            out += (-(c_lo + c_hi)).reshape(shape) * v
            up = [slice(None)] * self.dim
            dn = [slice(None)] * self.dim
            up[a] = slice(1, None)
            dn[a] = slice(None, -1)
            out[tuple(up)] += c_lo[1:].reshape(shape) * v[tuple(dn)]
            out[tuple(dn)] += c_hi[:-1].reshape(shape) * v[tuple(up)]
        return out

    def tridiag(self, a):  # pml.py:104-113
        c_lo, c_hi = self.couplings(a)
        m = c_lo.size
        T = np.zeros((m, m), dtype=np.complex128)
        i = np.arange(m)
        T[i, i] = -(c_lo + c_hi)
        T[i[1:], i[1:] - 1] = c_lo[1:]
        T[i[:-1], i[:-1] + 1] = c_hi[:-1]
        return T

    def to_sparse(self):  # pml.py:161-173
        eyes = [sp.identity(m, dtype=np.complex128, format="csr") for m in self.shape]
        total = None
        for a in range(self.dim):
            c_lo, c_hi = self.couplings(a)
            Ta = sp.diags([c_lo[1:], -(c_lo + c_hi), c_hi[:-1]], [-1, 0, 1], format="csr")
            fs = [eyes[b] if b != a else Ta for b in range(self.dim)]
            term = fs[0]
            for f in fs[1:]:
                term = sp.kron(term, f, format="csr")
            total = term if total is None else total + term
        k2 = np.broadcast_to(self.k2_on(self.lo, self.shape), self.shape).ravel()
        return (total + sp.diags(k2)).tocsr()

    def fingerprint_bytes(self):
        parts = [repr((self.shape, self.kappa2_kind, self.prob.spacing)).encode()]
        parts += [a.tobytes() for a in (*self.alpha_nodes, *self.alpha_faces)]
        if self.kappa2_kind == "const":
            parts.append(repr(self.kappa2).encode())
        elif self.kappa2_kind == "axis":
            parts += [repr(self.kappa2[0]).encode(), self.kappa2[1].tobytes()]
        else:
            parts.append(self.kappa2.tobytes())
        return b"".join(parts)


# ------------------------------------------------------ local solvers
_trsyl = get_lapack_funcs(("trsyl",), (np.zeros((1, 1), np.complex128),))[0]


def _sylv(A, B, Cm):  # subdomain.py:30-40
    Y, scale, info = _trsyl(A, B, Cm)
    assert info >= 0
    return Y / scale


class Separable:
    """Schur/Sylvester fast solver (subdomain.py:43-106)."""

    def __init__(self, op: Op):
        T = [op.tridiag(a) for a in range(op.dim)]
        if op.kappa2_kind == "axis":
            ax, vals = op.kappa2
            T[ax] += np.diag(vals.astype(np.complex128))
            k2 = 0.0
        else:
            k2 = complex(op.kappa2)
        last = op.dim - 1
        B_last = T[last].T + k2 * np.eye(op.shape[last], dtype=np.complex128)
        self.R1, self.Q1 = schur(T[0], output="complex")
        self.R2, self.Q2 = schur(B_last, output="complex")
        if op.dim == 3:
            self.R3, self.Q3 = schur(T[1], output="complex")
        self.dim = op.dim
        self.shape = op.shape

    def solve(self, rhs):
        if self.dim == 2:
            Cm = self.Q1.conj().T @ rhs @ self.Q2
            Y = _sylv(self.R1, self.R2, Cm)
            return np.ascontiguousarray(self.Q1 @ Y @ self.Q2.conj().T)
        Q1, R1, Q2, R2, Q3, R3 = self.Q1, self.R1, self.Q2, self.R2, self.Q3, self.R3
        Cm = np.einsum("ai,ijk->ajk", Q1.conj().T, rhs)
        Cm = np.einsum("kb,ajk->ajb", Q2, Cm)
        Cm = np.einsum("jc,ajb->acb", Q3.conj(), Cm)
        m = self.shape[1]
        Y = np.empty_like(Cm)
        eye = np.eye(R1.shape[0], dtype=np.complex128)
        for s in range(m - 1, -1, -1):
            r = Cm[:, s, :]
            if s < m - 1:
                r = r - np.einsum("c,acb->ab", R3[s, s + 1:], Y[:, s + 1:, :])
            Y[:, s, :] = _sylv(R1 + R3[s, s] * eye, R2, r)
        out = np.einsum("jc,acb->ajb", Q3, Y)
        out = np.einsum("kb,ajb->ajk", Q2.conj(), out)
        out = np.einsum("ia,ajk->ijk", Q1, out)
        return np.ascontiguousarray(out)


class SparseLU:
    """SuperLU on the window matrix (subdomain.py:109-133)."""

    def __init__(self, op: Op):
        self.shape = op.shape
        spec = "COLAMD" if op.dim == 2 else "MMD_AT_PLUS_A"
        self.lu = spla.splu(op.to_sparse().tocsc(), permc_spec=spec)

    def solve(self, rhs):
        return self.lu.solve(rhs.ravel().astype(np.complex128)).reshape(self.shape)


def factorize(op: Op, method="auto"):  # subdomain.py:139-146
    if method == "auto":
        method = "separable" if op.kappa2_kind != "full" else "splu"
    return Separable(op) if method == "separable" else SparseLU(op)


class Cache:  # subdomain.py:153-179 (fingerprint = raw coefficient bytes)
    def __init__(self, method="auto"):
        self.method = method
        self.store = {}
        self.factor_time = 0.0

    def get(self, op):
        key = op.fingerprint_bytes()
        f = self.store.get(key)
        if f is None:
            t = time.perf_counter()
            f = factorize(op, self.method)
            self.factor_time += time.perf_counter() - t
            self.store[key] = f
        return f


# ------------------------------------------------------- sweep rules
DEFAULT_2D = ((1, 1), (-1, 1), (1, -1), (-1, -1))  # ddm.py:36-40
DEFAULT_3D = ((1, 1, 1), (-1, 1, 1), (1, -1, 1), (-1, -1, 1),
              (1, 1, -1), (-1, 1, -1), (1, -1, -1), (-1, -1, -1))


def source_directions(dim):  # ddm.py:75-79
    return tuple(d for d in itertools.product((-1, 0, 1), repeat=dim) if any(d))


def similar(d1, d2, dim):  # transfer.py:63-67
    dot = sum(a * b for a, b in zip(d1, d2))
    return dot > 0 if dim == 2 else dot > 0 and all(a * b >= 0 for a, b in zip(d1, d2))


def rule_allows(src, gen, use, dim):  # transfer.py:76-87
    if not similar(src, use, dim):
        return False
    planes = ((0, 1),) if dim == 2 else ((0, 1), (0, 2), (1, 2))
    for ax in planes:
        s = [src[a] for a in ax]
        if sum(1 for c in s if c == 0) == 1 and all(gen[a] == -use[a] for a in ax):
            return False
    return True


def next_usable(src, gen_sweep, directions):  # transfer.py:90-97
    dim = len(src)
    for use in range(gen_sweep, len(directions) + 1):
        if rule_allows(src, directions[gen_sweep - 1], directions[use - 1], dim):
            return use
    return None


def sweep_step(idx, direction, counts):  # partition.py:209-217
    return 1 + sum((i - 1) if c == 1 else (n - i) for i, c, n in zip(idx, direction, counts))


def content_cuts(direction, parent):  # ddm.py:82-93
    out = {(a, -c) for a, c in enumerate(direction) if c}
    out |= {(a, s) for (a, s) in parent if direction[a] == 0}
    return frozenset(out)


def solve_cuts(arrivals, has_own):  # ddm.py:96-100
    if has_own or not arrivals:
        return frozenset()
    return frozenset.intersection(*arrivals)


def emits(direction, cuts):  # ddm.py:103-110
    return not any(c != 0 and (a, c) in cuts for a, c in enumerate(direction))


def _sl(lo, hi, ref_lo=None):
    if ref_lo is None:
        return tuple(slice(l, h + 1) for l, h in zip(lo, hi))
    return tuple(slice(l - r, h - r + 1) for l, h, r in zip(lo, hi, ref_lo))


def psi(prob, ops, idx, direction, v, rhs):  # transfer.py:100-155
    nb = tuple(i + c for i, c in zip(idx, direction))
    if any(not 1 <= i <= n for i, n in zip(nb, prob.part_counts)):
        return None
    d = prob.d
    slo, shi = prob.window(idx)
    nlo, nhi = prob.window(nb)
    lo, hi = [], []
    for a, c in enumerate(direction):
        bk = prob.breaks[a]
        i = idx[a]
        if c == 1:
            lo.append(bk[i]); hi.append(bk[i] + d)
        elif c == -1:
            lo.append(bk[i - 1] - d); hi.append(bk[i - 1])
        else:
            lo.append(max(slo[a], nlo[a])); hi.append(min(shi[a], nhi[a]))
    elo = [max(l - 1, s, n) for l, s, n in zip(lo, slo, nlo)]
    ehi = [min(h + 1, s, n) for h, s, n in zip(hi, shi, nhi)]
    eshape = tuple(h - l + 1 for l, h in zip(elo, ehi))
    weight = np.ones(eshape)
    order = 0
    for a, c in enumerate(direction):
        if c == 0:
            continue
        order += 1
        shape = [1] * prob.dim
        shape[a] = -1
        nodes = np.arange(elo[a], ehi[a] + 1)
        weight = weight * (1.0 - prob.beta_1d_nodes(a, c, idx[a], nodes).reshape(shape))
    w = (weight - 1.0) * v[_sl(elo, ehi, slo)]
    sign = 1.0 if order % 2 == 1 else -1.0
    lw = ops[nb].apply(w, tuple(elo))
    payload = sign * (rhs[_sl(lo, hi, slo)] + lw[_sl(lo, hi, elo)])
    return nb, (tuple(lo), tuple(hi)), payload


def ddm_apply(prob: Problem, ops, cache: Cache, f, directions=None, record=False,
              snapshot_at=()):
    """diagonal_sweep_solve restated (ddm.py:212-291) for one RHS.

    snapshot_at: (sweep, step) pairs (test hook); right after each such
    anti-diagonal step rep["snapshots"][(sweep, step)] = (u copy, pending),
    pending = {(use sweep, target, direction): (band lo, band hi, summed
    payload)} -- the state a per-step GPU check compares (the partial sum of
    _accumulate and the queued psi payloads)."""
    t0 = time.perf_counter()
    dim = prob.dim
    directions = directions or (DEFAULT_2D if dim == 2 else DEFAULT_3D)
    dirs = source_directions(dim)
    own = {}
    for idx in prob.subdomains:  # restrict_source (ddm.py:168-195)
        olo, ohi = prob.owned(idx)
        own[idx] = (olo, ohi, np.ascontiguousarray(f[_sl(olo, ohi)], dtype=np.complex128))
    queues = {}
    u = np.zeros(prob.counts, dtype=np.complex128)
    nsteps = sum(prob.part_counts) - dim + 1
    rep = {"solves": 0, "nonzero_solves": 0, "discarded_sources": 0, "events": []}
    for sweep, sd in enumerate(directions, 1):
        groups = {}
        for idx in prob.subdomains:
            groups.setdefault(sweep_step(idx, sd, prob.part_counts), []).append(idx)
        for step in range(1, nsteps + 1):
            for idx in sorted(groups.get(step, [])):
                wlo, whi = prob.window(idx)
                rhs = np.zeros(tuple(h - l + 1 for l, h in zip(wlo, whi)), dtype=np.complex128)
                arrivals = []
                has_own = False
                if sweep == 1:
                    olo, ohi, vals = own[idx]
                    has_own = bool(np.any(vals))
                    rhs[_sl(olo, ohi, wlo)] += vals
                consumed = 0
                for (blo, bhi, vals, cuts, _dv) in queues.pop((sweep, idx), []):
                    rhs[_sl(blo, bhi, wlo)] += vals
                    arrivals.append(cuts)
                    consumed += 1
                cuts = solve_cuts(arrivals, has_own)
                nonzero = bool(np.any(rhs))
                emitted = 0
                if nonzero:
                    ul = cache.get(ops[idx]).solve(rhs)
                    rep["nonzero_solves"] += 1
                    (slo, shi), beta = prob.beta00_support(idx)
                    u[_sl(slo, shi)] += beta * ul[_sl(slo, shi, wlo)]
                    for dvec in dirs:
                        if not emits(dvec, cuts):
                            continue
                        res = psi(prob, ops, idx, dvec, ul, rhs)
                        if res is None:
                            continue
                        target, (blo, bhi), payload = res
                        use = next_usable(dvec, sweep, directions)
                        if use is None:
                            rep["discarded_sources"] += 1
                        else:
                            queues.setdefault((use, target), []).append(
                                (blo, bhi, payload, content_cuts(dvec, cuts), dvec))
                            emitted += 1
                rep["solves"] += 1
                if record:
                    rep["events"].append({"sweep": sweep, "step": step, "subdomain": list(idx),
                                          "sources_consumed": consumed,
                                          "sources_emitted": emitted, "nonzero": nonzero})
            if (sweep, step) in snapshot_at:
                pending = {}
                for (use, target), entries in queues.items():
                    for (blo, bhi, vals, _c, dv) in entries:
                        key = (use, target, dv)
                        if key in pending:
                            pending[key] = (blo, bhi, pending[key][2] + vals)
                        else:
                            pending[key] = (blo, bhi, vals.copy())
                rep.setdefault("snapshots", {})[(sweep, step)] = (u.copy(), pending)
    assert not queues
    rep["wall_time"] = time.perf_counter() - t0
    return u, rep


def additive_apply(prob: Problem, ops, cache: Cache, f):
    """additive_ddm_solve restated (ddm.py:294-349) for one RHS: every step
    solves every subdomain; a target at step s gathers psi of each in-range
    source idx - c solved at level s - |c|_1 that emits towards it."""
    t0 = time.perf_counter()
    dim = prob.dim
    dirs = source_directions(dim)
    own = {}
    for idx in prob.subdomains:  # restrict_source (ddm.py:168-195)
        olo, ohi = prob.owned(idx)
        own[idx] = (olo, ohi, np.ascontiguousarray(f[_sl(olo, ohi)], dtype=np.complex128))
    u = np.zeros(prob.counts, dtype=np.complex128)
    total = sum(prob.part_counts) - dim + 1
    rep = {"solves": 0, "nonzero_solves": 0, "discarded_sources": 0, "first_nonzero_step": {}}
    history = {}
    for step in range(1, total + 1):
        current = {}
        for idx in sorted(prob.subdomains):
            wlo, whi = prob.window(idx)
            rhs = np.zeros(tuple(h - l + 1 for l, h in zip(wlo, whi)), dtype=np.complex128)
            arrivals = []
            has_own = False
            if step == 1:
                olo, ohi, vals = own[idx]
                has_own = bool(np.any(vals))
                rhs[_sl(olo, ohi, wlo)] += vals
            else:
                for dvec in dirs:
                    level = step - sum(abs(c) for c in dvec)
                    src = tuple(i - c for i, c in zip(idx, dvec))
                    if level < 1 or any(not 1 <= i <= n for i, n in zip(src, prob.part_counts)):
                        continue
                    entry = history.get(level, {}).get(src)
                    if entry is None or not emits(dvec, entry[2]):
                        continue
                    res = psi(prob, ops, src, dvec, entry[0], entry[1])
                    target, (blo, bhi), payload = res
                    rhs[_sl(blo, bhi, wlo)] += payload
                    arrivals.append(content_cuts(dvec, entry[2]))
            rep["solves"] += 1
            if np.any(rhs):
                ul = cache.get(ops[idx]).solve(rhs)
                rep["nonzero_solves"] += 1
                (slo, shi), beta = prob.beta00_support(idx)
                u[_sl(slo, shi)] += beta * ul[_sl(slo, shi, wlo)]
                current[idx] = (ul, rhs, solve_cuts(arrivals, has_own))
                rep["first_nonzero_step"].setdefault(idx, step)
            else:
                current[idx] = None
        history[step] = current
        history.pop(step - dim, None)
    rep["wall_time"] = time.perf_counter() - t0
    return u, rep


def gmres(apply_A, apply_M, b, tol=1e-6, restart=30, max_iter=200):
    """Right-preconditioned restarted GMRES restated (krylov.py:40-147)."""
    shape = b.shape
    b = np.asarray(b, dtype=np.complex128).ravel()
    norm_b = np.linalg.norm(b)
    x = np.zeros_like(b)
    rep = {"n_iter": 0, "converged": False, "residuals": []}
    if norm_b == 0.0:
        rep["converged"] = True
        rep["residuals"].append(0.0)
        return x.reshape(shape), rep
    A = lambda v: np.asarray(apply_A(v.reshape(shape)), dtype=np.complex128).ravel()
    M = lambda v: np.asarray(apply_M(v.reshape(shape)), dtype=np.complex128).ravel()
    residual = norm_b
    rep["residuals"].append(1.0)
    total = 0
    while total < max_iter and residual / norm_b > tol:
        r = b - A(x)
        beta = np.linalg.norm(r)
        m = min(restart, max_iter - total)
        V = np.zeros((m + 1, b.size), dtype=np.complex128)
        Z = np.zeros((m, b.size), dtype=np.complex128)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m, dtype=np.complex128)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        k_done = 0
        for k in range(m):
            Z[k] = M(V[k])
            w = A(Z[k]).copy()
            n0 = np.linalg.norm(w)
            for i in range(k + 1):
                H[i, k] = np.vdot(V[i], w)
                w -= H[i, k] * V[i]
            if np.linalg.norm(w) < 0.5 * n0:
                for i in range(k + 1):
                    c = np.vdot(V[i], w)
                    H[i, k] += c
                    w -= c * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            for i in range(k):
                hi = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -np.conj(sn[i]) * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = hi
            denom = np.hypot(abs(H[k, k]), abs(H[k + 1, k]))
            if denom == 0.0:
                k_done = k + 1
                break
            if H[k, k] == 0:
                cs[k] = 0.0
                sn[k] = np.conj(H[k + 1, k]) / abs(H[k + 1, k])
            else:
                cs[k] = abs(H[k, k]) / denom
                sn[k] = (H[k, k] / abs(H[k, k])) * np.conj(H[k + 1, k]) / denom
            H[k, k] = cs[k] * H[k, k] + sn[k] * H[k + 1, k]
            norm_w = H[k + 1, k].real
            H[k + 1, k] = 0.0
            g[k + 1] = -np.conj(sn[k]) * g[k]
            g[k] = cs[k] * g[k]
            k_done = k + 1
            total += 1
            residual = abs(g[k + 1])
            rep["n_iter"] = total
            rep["residuals"].append(residual / norm_b)
            if residual / norm_b <= tol or norm_w == 0.0:
                break
            V[k + 1] = w / norm_w
        if k_done:
            y = np.linalg.solve(np.triu(H[:k_done, :k_done]), g[:k_done])
            x = x + Z[:k_done].T @ y
        residual = np.linalg.norm(b - A(x))
        rep["residuals"][-1] = residual / norm_b
        if k_done == 0:
            break
    rep["converged"] = bool(residual / norm_b <= tol)
    return x.reshape(shape), rep


def gmres_ddm(prob: Problem, ops, gop: Op, cache: Cache, f, tol=1e-6, restart=30, max_iter=200):
    """The cli.py:78-97 gmres-ddm mode for one RHS."""
    return gmres(lambda v: gop.apply(v),
                 lambda v: ddm_apply(prob, ops, cache, v)[0], f, tol, restart, max_iter)
