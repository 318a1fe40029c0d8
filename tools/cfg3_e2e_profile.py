import sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve, gmres_batched
s = configs.spec(3); b = configs.build(s); f = configs.sources(s, b["grid"])
part, ops, gop = b["partition"], b["ops"], b["gop"]
cache = FactorizationCache()
full = part.grid.full_window()
f_pin = torch.from_numpy(f).pin_memory()
def step():
    x, _ = gmres_batched(lambda v: gop.apply(v, region=full),
                         lambda v: diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)[0].values,
                         f_pin, tol=1e-6)
    return x
for _ in range(2): step()
torch.cuda.synchronize()
t0 = time.perf_counter(); x = step(); torch.cuda.synchronize(); print("e2e step ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile(); pr.enable(); x = step(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
