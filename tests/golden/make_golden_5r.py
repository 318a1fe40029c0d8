#!/usr/bin/env python
"""Golden GMRES-DDM solution of config 5r (the oracle-feasible
stand-in for config 5), one RHS, produced by the REFERENCE package.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_5r.py
(takes ~5 minutes: 64 SuperLU factorizations + 5 GMRES iterations)
"""
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))
import diagsweep as R  # noqa: E402
from diagsweep.media import RasterModel  # noqa: E402

from paper_2002_05327_b200 import configs  # noqa: E402

s = configs.spec("5r")
b = configs.build(s)
g = b["grid"]
rg = R.make_grid(g.extents, g.counts)
rp = R.make_partition(rg, s.counts, s.d, s.pml)
prof = R.PmlProfile(s.pml, s.d, s.sigma_max, s.exponent)
model = RasterModel(tuple(s.interior), b["c"])
ops = R.build_operators(rp, prof, model, b["omega"])
gop = R.build_global_operator(rp, prof, model, b["omega"])
f = configs.sources(s, g)[0]
cache = R.FactorizationCache()
full = rg.full_window()
t0 = time.time()
x, rep = R.gmres(lambda v: gop.apply(v, region=full),
                 lambda v: R.diagonal_sweep_solve(v, rp, ops, cache, warn_collar=False)[0].values,
                 f, tol=1e-6, restart=30, max_iter=200)
print("5r gmres", rep.n_iter, rep.converged, time.time() - t0)
np.savez_compressed(HERE / "gmres_cfg5r.npz", x=x, residuals=np.array(rep.residuals),
                    n_iter=rep.n_iter, converged=rep.converged,
                    source_sha=hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest())
