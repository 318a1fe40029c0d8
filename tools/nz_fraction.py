import sys; sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200.ddm import SweepPlan, device_plan
for cfg in (2, 4):
    s = configs.spec(cfg); b = configs.build(s); f = configs.sources(s, b["grid"])
    part, ops = b["partition"], b["ops"]
    dp = device_plan(part, ops, FactorizationCache(), SweepPlan.default(part.dim), f.shape[0])
    fd = torch.from_numpy(f.reshape(f.shape[0], -1)).cuda()
    dp.apply(fd); torch.cuda.synchronize()
    c = dp.counters(f.shape[0])
    vnz = c["visit_nonzero"]
    print(cfg, "nonzero (visit,rhs) fraction", vnz.mean(), "visits with any nonzero", (vnz.sum(-1) > 0).mean(), "per sweep", vnz.mean(axis=(1, 2)))
