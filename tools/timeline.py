"""Kernel timeline of one DDM application under CUDA-graph replay (CUPTI via
torch.profiler): per stream the kernels' start / duration / gap, and how much
of the step has 0, 1 or >= 2 kernels running.

usage: python tools/timeline.py [config] [groups] [out.json]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200.ddm import SweepPlan, device_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
cfg = int(cfg) if cfg.isdigit() else cfg
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 2
out = sys.argv[3] if len(sys.argv) > 3 else None
s = configs.spec(cfg)
b = configs.build(s)
f = configs.sources(s, b["grid"])
part, ops = b["partition"], b["ops"]
cache = FactorizationCache()
dp = device_plan(part, ops, cache, SweepPlan.default(part.dim), f.shape[0], grouped=groups > 1)
fd = torch.from_numpy(f.reshape(f.shape[0], -1)).cuda()
for _ in range(4):
    dp.apply(fd)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    dp.apply(fd)
    torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0:
        ev.append({"name": e.name[:40], "start": e.time_range.start, "dur": e.time_range.end - e.time_range.start,
                   "stream": getattr(e, "stream", None) if hasattr(e, "stream") else None})
ev.sort(key=lambda x: x["start"])
t0 = ev[0]["start"]
t1 = max(e["start"] + e["dur"] for e in ev)
print(f"{len(ev)} kernels, span {t1 - t0:.1f} us")
# per kernel-name totals
tot = {}
for e in ev:
    a = tot.setdefault(e["name"], [0, 0.0])
    a[0] += 1
    a[1] += e["dur"]
for k, (n, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"  {k:42s} n={n:4d} total {d:8.1f} us  avg {d / n:6.2f}")
# concurrency histogram by sweep line
pts = []
for e in ev:
    pts.append((e["start"], 1))
    pts.append((e["start"] + e["dur"], -1))
pts.sort()
hist = {}
lvl, last = 0, pts[0][0]
for t, d in pts:
    hist[lvl] = hist.get(lvl, 0.0) + (t - last)
    lvl += d
    last = t
print("concurrency (kernels running -> us):", {k: round(v, 1) for k, v in sorted(hist.items())})
if out:
    for e in ev:
        e["start"] -= t0
    Path(out).write_text(json.dumps(ev))
