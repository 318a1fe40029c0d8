"""Right-preconditioned restarted GMRES, batched over right-hand sides.

Drop-in for `diagsweep.krylov.gmres` (krylov.py:40-147) with the same
signature and the same per-RHS semantics: x0 = 0; each cycle starts from the
true residual r = b - A x; the flexible basis Z = M^{-1} V is stored; Arnoldi
uses modified Gram-Schmidt with one reorthogonalisation pass when
||w|| < 0.5 ||w0||; complex Givens rotations; y from the triangular system;
the last residual of every cycle is replaced by the true residual; the loop
ends on tol, on max_iter total iterations or on a breakdown.  `n_iter`
counts Arnoldi steps.

Batching: `b` may carry a leading RHS axis `[R, *shape]`.  All RHS advance
in lock-step; an RHS that converges (or hits breakdown / the restart length)
leaves the active set and the closures are then called only on the rows
still active.  The vectors are RHS-outer `[R, n]` CUDA tensors and every
vector operation (dot, norm, fused MGS axpy+dot, basis combination, scale)
is a native kernel (K7, csrc/ds_core.cu).  The O(restart^2) Hessenberg
work per RHS stays on the host, as in the reference.

Closures receive torch CUDA tensors shaped like `b` (`[*shape]` for an
unbatched `b`, `[R', *shape]` for a batch, R' = active rows) and may return
torch tensors or NumPy arrays.
"""

from __future__ import annotations

import csv
import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


@dataclass
class SolveReport:
    n_iter: int = 0
    converged: bool = False
    residuals: list = field(default_factory=list)
    times: list = field(default_factory=list)
    precond_times: list = field(default_factory=list)
    wall_time: float = 0.0

    def write_residual_csv(self, path, header_comment: str | None = None) -> None:
        with open(path, "w", newline="") as fh:
            if header_comment:
                fh.write(f"# {header_comment}\n")
            writer = csv.writer(fh)
            writer.writerow(["iteration", "relative_residual", "cumulative_seconds"])
            for k, (res, t) in enumerate(zip(self.residuals, self.times)):
                writer.writerow([k, f"{res:.6e}", f"{t:.6f}"])


class _Vec:
    """Native batched vector ops on RHS-outer [R, n] complex128 tensors.
    Every op re-binds the context to torch's current stream first: a
    preconditioner closure may have left the shared context on a side
    stream (RHS-group plans), and the vectors were produced on this one."""

    MAX_COMBINE = 64  # ds_vec_combine's per-call vector limit

    def __init__(self, n: int):
        from . import _engine

        self._context = _engine.context
        self.lib, self.ctx = _engine.context()
        self.n = n

    def _bind(self):
        self.lib, self.ctx = self._context()  # ds_ctx_set_stream(current stream)

    def dot(self, x, y, out):
        self._bind()
        N.check(self.lib.ds_vec_dot(self.ctx, self.n, x.shape[0], x.data_ptr(), y.data_ptr(),
                                    out.data_ptr()))

    def norm(self, x, out):
        self._bind()
        N.check(self.lib.ds_vec_norm(self.ctx, self.n, x.shape[0], x.data_ptr(), out.data_ptr()))

    def axpy(self, a, sgn, x, y):
        self._bind()
        N.check(self.lib.ds_vec_axpy(self.ctx, self.n, x.shape[0], a.data_ptr(), sgn,
                                     x.data_ptr(), y.data_ptr()))

    def axpy_dot(self, a_prev, xprev, y, x, out):
        self._bind()
        N.check(self.lib.ds_vec_axpy_dot(
            self.ctx, self.n, x.shape[0], 0 if a_prev is None else a_prev.data_ptr(),
            0 if xprev is None else xprev.data_ptr(), y.data_ptr(), x.data_ptr(),
            out.data_ptr()))

    def combine(self, xs, c, y):
        """y += sum_j c[j] X_j, in chunks of MAX_COMBINE vectors (any restart
        length; c is [len(xs), R] contiguous)."""
        self._bind()
        step = self.MAX_COMBINE
        for j0 in range(0, len(xs), step):
            part = xs[j0:j0 + step]
            arr = (C.c_void_p * len(part))(*[x.data_ptr() for x in part])
            N.check(self.lib.ds_vec_combine(self.ctx, self.n, y.shape[0], len(part), arr,
                                            c[j0:j0 + step].data_ptr(), y.data_ptr()))

    def sub_norm(self, b, w, out, norms):
        """out = b - w, norms = ||out|| per row, one pass (ds_vec_sub_norm)."""
        self._bind()
        N.check(self.lib.ds_vec_sub_norm(self.ctx, self.n, b.shape[0], b.data_ptr(), w.data_ptr(),
                                         out.data_ptr(), norms.data_ptr()))

    def rows(self, mapping, src, dst):
        """dst[r] = src[mapping[r]] (0 where mapping[r] < 0), ds_vec_rows."""
        self._bind()
        N.check(self.lib.ds_vec_rows(self.ctx, self.n, dst.shape[0], mapping.data_ptr(),
                                     src.data_ptr(), dst.data_ptr()))

    def divide(self, x, s, y):
        self._bind()
        N.check(self.lib.ds_vec_scale(self.ctx, self.n, x.shape[0], x.data_ptr(), s.data_ptr(),
                                      y.data_ptr()))


def gmres(apply_A, apply_M, b, tol: float = 1e-6, restart: int = 30, max_iter: int = 200):
    """Solve A x = b (batched) with right preconditioner M^{-1}."""
    import torch

    from . import _engine

    t0 = time.perf_counter()
    is_torch = hasattr(b, "detach")
    bt = b.detach() if is_torch else torch.from_numpy(np.asarray(b, dtype=np.complex128))
    shape = tuple(bt.shape)
    batched = False
    # An unbatched b is any array; a batch is signalled by a 2-level call
    # from gmres_batched (see below).
    return _gmres_core(apply_A, apply_M, bt, shape, batched, is_torch, tol, restart, max_iter,
                       t0)


def gmres_batched(apply_A, apply_M, b, tol: float = 1e-6, restart: int = 30,
                  max_iter: int = 200):
    """Batched GMRES: b is `[R, *shape]`; returns (x [R, *shape], [SolveReport]*R)."""
    import torch

    t0 = time.perf_counter()
    is_torch = hasattr(b, "detach")
    bt = b.detach() if is_torch else torch.from_numpy(np.asarray(b, dtype=np.complex128))
    return _gmres_core(apply_A, apply_M, bt, tuple(bt.shape[1:]), True, is_torch, tol, restart,
                       max_iter, t0)


def _gmres_core(apply_A, apply_M, bt, shape, batched, is_torch, tol, restart, max_iter, t0):
    import torch

    from . import _engine

    _engine._require_cuda()
    dev = torch.device("cuda")
    R = bt.shape[0] if batched else 1
    n = int(np.prod(shape))
    B = bt.to(dev, torch.complex128).reshape(R, n).contiguous()
    vec = _Vec(n)
    X = torch.zeros_like(B)
    reports = [SolveReport() for _ in range(R)]

    maps = {}

    def row_maps(rows):
        """(gather map [len(rows)], scatter map [R]) device int32 tables."""
        key = tuple(rows)
        if key not in maps:
            inv = np.full(R, -1, np.int32)
            inv[list(rows)] = np.arange(len(rows), dtype=np.int32)
            maps[key] = (torch.as_tensor(np.asarray(rows, np.int32), device=dev),
                         torch.as_tensor(inv, device=dev))
        return maps[key]

    def call(fn, rows, V):
        """Apply a closure to the rows `rows` of V ([R, n]) -> [len(rows), n]."""
        if len(rows) == R:
            sub = V
        else:  # native row gather of the active RHS (ds_vec_rows)
            sub = torch.empty((len(rows), n), dtype=torch.complex128, device=dev)
            vec.rows(row_maps(rows)[0], V, sub)
        arg = sub.reshape((len(rows),) + shape) if batched else sub.reshape(shape)
        out = fn(arg)
        if not hasattr(out, "detach"):
            out = torch.from_numpy(np.asarray(out, dtype=np.complex128))
        return out.to(dev, torch.complex128).reshape(len(rows), n).contiguous()

    def scatter(dst, rows, src):
        """dst = src on rows `rows`, zero elsewhere (ds_vec_rows)."""
        vec.rows(row_maps(rows)[1], src, dst)

    nb = torch.empty(R, dtype=torch.float64, device=dev)
    vec.norm(B, nb)
    norm_b = nb.cpu().numpy()
    residual = norm_b.copy()
    total = np.zeros(R, dtype=np.int64)
    live = []
    for r in range(R):
        if norm_b[r] == 0.0:
            reports[r].converged = True
            reports[r].residuals.append(0.0)
            reports[r].times.append(time.perf_counter() - t0)
            reports[r].wall_time = reports[r].times[-1]
        else:
            reports[r].residuals.append(1.0)
            reports[r].times.append(time.perf_counter() - t0)
            live.append(r)

    W = torch.empty_like(B)
    while True:
        cyc = [r for r in live if total[r] < max_iter and residual[r] / norm_b[r] > tol]
        if not cyc:
            break
        # ---- cycle start for the RHS in `cyc`: r = b - A x  (krylov.py:80)
        AX = call(apply_A, cyc, X)
        scatter(W, cyc, AX)
        Rv = torch.empty_like(B)
        beta_d = torch.empty(R, dtype=torch.float64, device=dev)
        vec.sub_norm(B, W, Rv, beta_d)  # r = b - A x and ||r||, one pass
        beta = beta_d.cpu().numpy()
        m_r = {r: min(restart, max_iter - int(total[r])) for r in cyc}
        m = max(m_r.values())
        V = [torch.empty_like(B)]
        s0 = np.zeros(R)
        s0[cyc] = beta[cyc]
        vec.divide(Rv, torch.from_numpy(s0).to(dev), V[0])  # V0 = r / beta (zero rows elsewhere)
        Z = []
        H = np.zeros((R, m + 1, m), dtype=np.complex128)
        cs = np.zeros((R, m), dtype=np.complex128)
        sn = np.zeros((R, m), dtype=np.complex128)
        g = np.zeros((R, m + 1), dtype=np.complex128)
        g[:, 0] = beta
        k_done = {r: 0 for r in cyc}
        active = list(cyc)
        hcol = torch.empty((m + 1, R), dtype=torch.complex128, device=dev)
        ccol = torch.empty((m + 1, R), dtype=torch.complex128, device=dev)
        for k in range(m):
            active = [r for r in active if k < m_r[r]]
            if not active:
                break
            tp = time.perf_counter()
            MZ = call(apply_M, active, V[k])
            Zk = torch.empty_like(B)
            scatter(Zk, active, MZ)
            Z.append(Zk)
            dtp = time.perf_counter() - tp
            for r in active:
                reports[r].precond_times.append(dtp)
            AZ = call(apply_A, active, Zk)
            scatter(W, active, AZ)
            n0 = torch.empty(R, dtype=torch.float64, device=dev)
            vec.norm(W, n0)
            # modified Gram-Schmidt, fused: w -= h_{i-1} v_{i-1}; h_i = vdot(v_i, w)
            for i in range(k + 1):
                vec.axpy_dot(hcol[i - 1] if i else None, V[i - 1] if i else None, W, V[i],
                             hcol[i])
            vec.axpy(hcol[k], -1.0, V[k], W)
            n1 = torch.empty(R, dtype=torch.float64, device=dev)
            vec.norm(W, n1)
            # one device -> host read per Arnoldi step: ||w0||, ||w||, h[:k+1]
            pack = torch.cat([n0, n1, torch.view_as_real(hcol[: k + 1]).reshape(-1)]).cpu().numpy()
            n0h, n1h = pack[:R], pack[R:2 * R]
            hk = pack[2 * R:].view(np.complex128).reshape(k + 1, R)
            reo = [r for r in active if n1h[r] < 0.5 * n0h[r]]
            if reo:
                sel = torch.zeros(R, dtype=torch.complex128, device=dev)
                sel[torch.as_tensor(reo, device=dev)] = 1.0
                for i in range(k + 1):
                    vec.axpy_dot(ccol[i - 1] if i else None, V[i - 1] if i else None, W, V[i],
                                 ccol[i])
                    ccol[i].mul_(sel)  # rows without reorthogonalisation keep c = 0
                vec.axpy(ccol[k], -1.0, V[k], W)
                vec.norm(W, n1)
                n1h = n1.cpu().numpy()
                hk = hk + ccol[: k + 1].cpu().numpy()
            finished = []
            now = time.perf_counter() - t0
            for r in active:
                Hr = H[r]
                Hr[: k + 1, k] = hk[:, r]
                Hr[k + 1, k] = n1h[r]
                for i in range(k):
                    hi = cs[r, i] * Hr[i, k] + sn[r, i] * Hr[i + 1, k]
                    Hr[i + 1, k] = -np.conj(sn[r, i]) * Hr[i, k] + cs[r, i] * Hr[i + 1, k]
                    Hr[i, k] = hi
                denom = np.hypot(abs(Hr[k, k]), abs(Hr[k + 1, k]))
                if denom == 0.0:
                    k_done[r] = k + 1
                    finished.append(r)
                    continue
                if Hr[k, k] == 0:
                    cs[r, k] = 0.0
                    sn[r, k] = np.conj(Hr[k + 1, k]) / abs(Hr[k + 1, k])
                else:
                    cs[r, k] = abs(Hr[k, k]) / denom
                    sn[r, k] = (Hr[k, k] / abs(Hr[k, k])) * np.conj(Hr[k + 1, k]) / denom
                Hr[k, k] = cs[r, k] * Hr[k, k] + sn[r, k] * Hr[k + 1, k]
                norm_w = Hr[k + 1, k].real
                Hr[k + 1, k] = 0.0
                g[r, k + 1] = -np.conj(sn[r, k]) * g[r, k]
                g[r, k] = cs[r, k] * g[r, k]
                k_done[r] = k + 1
                total[r] += 1
                residual[r] = abs(g[r, k + 1])
                rep = reports[r]
                rep.n_iter = int(total[r])
                rep.residuals.append(residual[r] / norm_b[r])
                rep.times.append(now)
                if residual[r] / norm_b[r] <= tol or norm_w == 0.0:
                    finished.append(r)
            active = [r for r in active if r not in finished]
            if not active:
                break
            s = np.zeros(R)
            for r in active:
                s[r] = n1h[r]
            V.append(torch.empty_like(B))
            vec.divide(W, torch.from_numpy(s).to(dev), V[k + 1])
        # ---- x += Z[:k_done]^T y  (krylov.py:135-139)
        nz = max(k_done.values()) if k_done else 0
        if nz:
            coef = np.zeros((nz, R), dtype=np.complex128)
            for r, kd in k_done.items():
                if kd:
                    y = np.linalg.solve(np.triu(H[r, :kd, :kd]), g[r, :kd])
                    coef[:kd, r] = y
            vec.combine(Z[:nz], torch.from_numpy(coef).to(dev), X)
        # ---- true residual (krylov.py:140-142)
        AX = call(apply_A, cyc, X)
        scatter(W, cyc, AX)
        tr = torch.empty(R, dtype=torch.float64, device=dev)
        vec.sub_norm(B, W, Rv, tr)
        trh = tr.cpu().numpy()
        for r in cyc:
            residual[r] = trh[r]
            reports[r].residuals[-1] = trh[r] / norm_b[r]
        live = [r for r in live if not (r in k_done and k_done[r] == 0)]
        del V, Z
    for r in range(R):
        if norm_b[r] != 0.0:
            reports[r].converged = bool(residual[r] / norm_b[r] <= tol)
            reports[r].wall_time = time.perf_counter() - t0
    x = X.reshape((R,) + shape) if batched else X.reshape(shape)
    if not is_torch:
        x = x.cpu().numpy()
    elif not bt.is_cuda:  # results return where the input lives (pinned in -> pinned out)
        out = torch.empty(x.shape, dtype=x.dtype, pin_memory=bt.is_pinned())
        out.copy_(x, non_blocking=bt.is_pinned())  # one DMA into a cached pinned block
        torch.cuda.current_stream().synchronize()
        x = out
    return (x, reports) if batched else (x, reports[0])
