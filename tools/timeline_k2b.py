"""CUPTI kernel timeline of one batched window factorization of config 5
(K2b): time per kernel class and how many kernels run concurrently.

usage: python tools/timeline_k2b.py [windows]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2002_05327_b200 import _engine, configs

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = configs.spec(5)
b = configs.build(s)
ops = [b["ops"][i] for i in b["partition"].subdomains()]
pool = _engine.FactorPool(ops, k)
pool.load(0, 0)  # warm-up (attributes, allocations)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    pool.load_many([(i, q) for q, i in enumerate(range(k, 2 * k))])
    torch.cuda.synchronize()
ev = [(e.time_range.start, e.time_range.end, e.name[:40]) for e in prof.events()
      if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0]
ev.sort()
t0, t1 = ev[0][0], max(e[1] for e in ev)
print(f"{k} windows, {len(ev)} kernels, span {(t1 - t0) / 1e3:.1f} ms")
tot = {}
for a, bb, n in ev:
    x = tot.setdefault(n, [0, 0.0])
    x[0] += 1
    x[1] += bb - a
for n, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"  {n:42s} n={c:6d} total {d / 1e3:9.1f} ms  avg {d / c:8.1f} us")
pts = sorted([(a, 1) for a, _, _ in ev] + [(bb, -1) for _, bb, _ in ev])
hist, lvl, last = {}, 0, pts[0][0]
for t, d in pts:
    hist[lvl] = hist.get(lvl, 0.0) + (t - last)
    lvl += d
    last = t
print("concurrency (kernels running -> ms):", {kk: round(v / 1e3, 1) for kk, v in sorted(hist.items())})
