"""Runs a few DDM applications of one config (for ncu / compute-sanitizer).

usage: python tools/profile_step.py [config] [applications]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200.ddm import SweepPlan, device_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
cfg = int(cfg) if cfg.isdigit() else cfg
napp = int(sys.argv[2]) if len(sys.argv) > 2 else 2
s = configs.spec(cfg)
b = configs.build(s)
f = configs.sources(s, b["grid"])
part, ops = b["partition"], b["ops"]
cache = FactorizationCache(share_translates=(part.dim == 3 and s.medium == "constant"))
dp = device_plan(part, ops, cache, SweepPlan.default(part.dim), f.shape[0])
fd = torch.from_numpy(f.reshape(f.shape[0], -1)).cuda()
for _ in range(napp):
    u, _ = dp.apply(fd)
torch.cuda.synchronize()
print("ok", float(torch.linalg.vector_norm(u)))
