import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200 import ddm
s = configs.spec(2); b = configs.build(s); f = configs.sources(s, b["grid"])
part, ops = b["partition"], b["ops"]
R = f.shape[0]
cache = FactorizationCache()
fh = torch.from_numpy(f.reshape(R, -1)).pin_memory(); uh = torch.empty_like(fh).pin_memory()
for grouped in (False, True):
    dp = ddm.device_plan(part, ops, cache, ddm.SweepPlan.default(2), R, grouped=grouped)
    for _ in range(3): dp.apply_host(fh, uh)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20): dp.apply_host(fh, uh)
    dt = (time.perf_counter() - t) / 20
    print("grouped" if grouped else "single", "apply_host ms %.3f" % (dt * 1e3), flush=True)
