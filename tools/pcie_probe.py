"""Pinned host <-> device copy rates for the config-2 batch size (48 MB)."""
import time
import torch
n = 16 * 433 * 433
h = torch.empty(n, dtype=torch.complex128, pin_memory=True)
d = torch.empty(n, dtype=torch.complex128, device="cuda")
h2 = torch.empty(n, dtype=torch.complex128, pin_memory=True)
d2 = torch.empty(n, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    for _ in range(3): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
    print(name, f"{dt*1e3:.3f} ms  {h.numel()*16/dt/1e9:.1f} GB/s")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
print("both", f"{dt*1e3:.3f} ms")
