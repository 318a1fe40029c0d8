"""Timeline of the pinned-host path (diagonal_sweep_solve on a pinned batch,
ds_ddm_apply_host): kernels and copies of one call (CUPTI via
torch.profiler) and the host wall clock around it.

usage: python tools/timeline_e2e.py [config]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
cfg = int(cfg) if cfg.isdigit() else cfg
s = configs.spec(cfg)
b = configs.build(s)
f = torch.from_numpy(configs.sources(s, b["grid"])).pin_memory()
part, ops = b["partition"], b["ops"]
cache = FactorizationCache()
for _ in range(4):
    diagonal_sweep_solve(f, part, ops, cache, warn_collar=False)
torch.cuda.synchronize()
walls = []
for _ in range(10):
    t0 = time.perf_counter()
    diagonal_sweep_solve(f, part, ops, cache, warn_collar=False)
    walls.append((time.perf_counter() - t0) * 1e3)
print("wall ms per call (no profiler):", [round(w, 3) for w in walls])
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    diagonal_sweep_solve(f, part, ops, cache, warn_collar=False)
    wall = (time.perf_counter() - t0) * 1e3
print(f"wall ms under the profiler: {wall:.3f}")
ev = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0:
        ev.append((e.time_range.start, e.time_range.end, e.name[:28]))
ev.sort()
t0 = ev[0][0]
kern = [e for e in ev if "Memcpy" not in e[2] and "Memset" not in e[2]]
h2d = [e for e in ev if "HtoD" in e[2]]
d2h = [e for e in ev if "DtoH" in e[2]]
print(f"{len(ev)} device activities; span {ev[-1][1] - t0:.0f} us")
if h2d:
    print(f"H2D: {len(h2d)} copies, first start {h2d[0][0] - t0:.0f}, last end {h2d[-1][1] - t0:.0f}, "
          f"busy {sum(b - a for a, b, _ in h2d):.0f} us")
if d2h:
    print(f"D2H: {len(d2h)} copies, first start {d2h[0][0] - t0:.0f}, last end {max(b for _, b, _ in d2h) - t0:.0f}, "
          f"busy {sum(b - a for a, b, _ in d2h):.0f} us")
asm = [e for e in kern if "k_assemble" in e[2]]
print("k_assemble starts (us):", [round(e[0] - t0) for e in asm[:16]], "...", [round(e[0] - t0) for e in asm[-4:]])
print(f"last kernel end {max(b for _, b, _ in kern) - t0:.0f} us")
