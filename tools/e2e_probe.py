import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve
from paper_2002_05327_b200 import _engine, ddm
s = configs.spec(2); b = configs.build(s); f = configs.sources(s, b["grid"])
part, ops = b["partition"], b["ops"]
cache = FactorizationCache()
f_pin = torch.from_numpy(f).pin_memory()
for _ in range(3):
    diagonal_sweep_solve(f_pin, part, ops, cache, warn_collar=False)
torch.cuda.synchronize()
T = {}
def tic(k, t0): T[k] = T.get(k, 0) + time.perf_counter() - t0
for _ in range(10):
    t0 = time.perf_counter(); fdev, kind, batched = _engine.to_device_batch(f_pin, part.grid.counts); torch.cuda.synchronize(); tic("h2d", t0)
    t0 = time.perf_counter(); dp = ddm.device_plan(part, ops, cache, None, 16); u, _ = dp.apply(fdev.reshape(16, -1)); torch.cuda.synchronize(); tic("apply", t0)
    t0 = time.perf_counter(); ddm._reports(dp, 16, ddm.SweepPlan.default(2), part, False, False); tic("reports", t0)
    t0 = time.perf_counter(); _engine.from_device_batch(u, kind, batched); torch.cuda.synchronize(); tic("d2h", t0)
    t0 = time.perf_counter(); diagonal_sweep_solve(f_pin, part, ops, cache, warn_collar=False); torch.cuda.synchronize(); tic("full", t0)
print({k: round(v * 100, 2) for k, v in T.items()}, "ms each")
