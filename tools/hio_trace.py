import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200 import ddm
s = configs.spec(2); b = configs.build(s); f = configs.sources(s, b["grid"])
part, ops = b["partition"], b["ops"]
R = f.shape[0]
dp = ddm.device_plan(part, ops, FactorizationCache(), ddm.SweepPlan.default(2), R)
fh = torch.from_numpy(f.reshape(R, -1)).pin_memory(); uh = torch.empty_like(fh).pin_memory()
dp.set_profiling(False)
from paper_2002_05327_b200 import _native as N
lib = N.load_library()
lib.ds_ddm_enable_graph(None, dp.handle, 0)
for i in range(4):
    if i == 3: os.environ["X"] = "1"
    dp.apply_host(fh, uh)
