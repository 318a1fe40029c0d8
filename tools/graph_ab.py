"""A/B of the DDM application with and without CUDA-graph replay (config 2)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200.ddm import SweepPlan, device_plan

s = configs.spec(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
b = configs.build(s)
f = configs.sources(s, b["grid"])
cache = FactorizationCache()
dp = device_plan(b["partition"], b["ops"], cache, SweepPlan.default(b["partition"].dim), f.shape[0])
fd = torch.from_numpy(f.reshape(f.shape[0], -1)).cuda()
for graph in (False, True):
    dp.enable_graph(graph)
    for _ in range(3):
        dp.apply(fd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        u, _ = dp.apply(fd)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"graph={graph}: {ms:.2f} ms/app  {f.shape[0] / ms * 1e3:.1f} RHS/s")
