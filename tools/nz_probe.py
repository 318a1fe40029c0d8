"""Which visit's exact-zero flag differs between the GPU and the oracle (config 2, one RHS)?"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]
from oracle import ds_oracle as O
from paper_2002_05327_b200 import configs, diagonal_sweep_solve, FactorizationCache
import torch

s = configs.spec(2); b = configs.build(s)
f = configs.sources(s, b["grid"])
prob = O.Problem(**configs.oracle_problem(s, b)); oops = prob.operators()
r = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for variant in ("single", "batch16-numpy", "batch16-torch"):
    if variant == "single":
        u, rep = diagonal_sweep_solve(f[r], b["partition"], b["ops"], FactorizationCache(), record_events=True, warn_collar=False)
    elif variant == "batch16-numpy":
        u, reps = diagonal_sweep_solve(f, b["partition"], b["ops"], FactorizationCache(), record_events=True, warn_collar=False); rep = reps[r]
    else:
        u, reps = diagonal_sweep_solve(torch.from_numpy(f).cuda(), b["partition"], b["ops"], FactorizationCache(), record_events=True, warn_collar=False); rep = reps[r]
    print(variant, "nonzero", rep.nonzero_solves)
ref, orep = O.ddm_apply(prob, oops, O.Cache(), f[r], record=True)
print("oracle nonzero", orep["nonzero_solves"])
for e1, e2 in zip(rep.events, orep["events"]):
    if e1 != e2:
        print("GPU", e1); print("ORA", e2)
# magnitude of the owned source per subdomain
for idx in sorted(b["ops"]):
    olo, ohi = prob.owned(idx)
    vals = f[r][tuple(slice(l, h + 1) for l, h in zip(olo, ohi))]
    mx = np.abs(vals).max()
    if 0 < mx < 1e-250:
        print("tiny own source", idx, mx)
