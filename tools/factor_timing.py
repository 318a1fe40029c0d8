"""Factorization time of config N (cache.prepare, CUDA events), 3 repeats."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_05327_b200 import FactorizationCache, configs

s = configs.spec(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
b = configs.build(s)
part, ops = b["partition"], b["ops"]
for rep in range(3):
    cache = FactorizationCache()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    cache.prepare([ops[i] for i in part.subdomains()])
    e1.record()
    torch.cuda.synchronize()
    print(f"factor: {e0.elapsed_time(e1):.1f} ms (wall {1e3 * (time.perf_counter() - t0):.1f} ms)")
