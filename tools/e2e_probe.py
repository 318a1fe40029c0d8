"""Breakdown of one end-to-end diagonal_sweep_solve call (config 2, pinned
host sources): device-resident apply, host-buffer apply, report read-back,
whole API call.  usage: python tools/e2e_probe.py [config]"""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve
from paper_2002_05327_b200 import _engine, ddm
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = configs.spec(cfg); b = configs.build(s); f = configs.sources(s, b["grid"])
part, ops = b["partition"], b["ops"]
R = f.shape[0]
cache = FactorizationCache()
f_pin = torch.from_numpy(f).pin_memory()
f_dev = f_pin.cuda().reshape(R, -1)
u_pin = torch.empty(f_dev.shape, dtype=torch.complex128, pin_memory=True)
dp = ddm.device_plan(part, ops, cache, ddm.SweepPlan.default(part.dim), R)
for _ in range(3):
    diagonal_sweep_solve(f_pin, part, ops, cache, warn_collar=False)
    dp.apply(f_dev)
    dp.apply_host(f_pin.reshape(R, -1), u_pin)
torch.cuda.synchronize()
T = {}
def tic(k, t0): T[k] = T.get(k, 0) + time.perf_counter() - t0
n = 10
for _ in range(n):
    t0 = time.perf_counter(); dp.apply(f_dev); torch.cuda.synchronize(); tic("apply_device", t0)
    t0 = time.perf_counter(); dp.apply_host(f_pin.reshape(R, -1), u_pin); tic("apply_host", t0)
    t0 = time.perf_counter(); ddm._reports(dp, R, ddm.SweepPlan.default(part.dim), part, False, False); tic("reports", t0)
    t0 = time.perf_counter(); ddm.device_plan(part, ops, cache, ddm.SweepPlan.default(part.dim), R); tic("plan_lookup", t0)
    t0 = time.perf_counter(); torch.empty(f_dev.shape, dtype=torch.complex128, pin_memory=True); tic("pinned_alloc", t0)
    t0 = time.perf_counter(); diagonal_sweep_solve(f_pin, part, ops, cache, warn_collar=False); tic("api_call", t0)
print({k: round(v * 1e3 / n, 3) for k, v in T.items()}, "ms each")
