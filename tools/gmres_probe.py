"""Decompose the GPU-vs-oracle GMRES solution difference (raster mini problem):
x_h = oracle GMRES driven by the GPU operator / preconditioner, so
|x_gpu - x_h| is the Krylov implementation and |x_h - x_oracle| the operators."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
from oracle import ds_oracle as O
from paper_2002_05327_b200 import configs, diagonal_sweep_solve, gmres_batched, FactorizationCache
from test_gpu_parity import mini_raster_spec

def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))

for name, s in [("mini", mini_raster_spec()), ("5r", configs.spec("5r"))]:
    b = configs.build(s)
    prob = O.Problem(**configs.oracle_problem(s, b)); ops = prob.operators(); gop = prob.global_operator()
    f = configs.sources(s, b["grid"])[:2]
    part, gops, ggop = b["partition"], b["ops"], b["gop"]
    cache = FactorizationCache(); full = part.grid.full_window()
    A = lambda v: ggop.apply(v, region=full)
    M = lambda v: diagonal_sweep_solve(v, part, gops, cache, warn_collar=False)[0].values
    xg, reps = gmres_batched(A, M, f, tol=1e-6)
    oc = O.Cache()
    for r in range(f.shape[0]):
        xo, ro = O.gmres_ddm(prob, ops, gop, oc, f[r])
        xh, rh = O.gmres(lambda v: np.asarray(A(v)), lambda v: np.asarray(M(v)), f[r])
        uo = O.ddm_apply(prob, ops, oc, f[r])[0]
        ug = M(f[r])
        print(f"{name} rhs{r}: it gpu/hyb/oracle {reps[r].n_iter}/{rh['n_iter']}/{ro['n_iter']} "
              f"x_gpu-x_or {rel(xg[r], xo):.3e} x_gpu-x_hyb {rel(xg[r], xh):.3e} "
              f"x_hyb-x_or {rel(xh, xo):.3e} u_ddm {rel(ug, uo):.3e} "
              f"Au {rel(A(f[r]), gop.apply(f[r])):.3e}", flush=True)
