"""Small end-to-end run for compute-sanitizer: config-1 geometry, modal and
block-LU backends, device path (grouped), pinned host path, 3D mini modal."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve
s = configs.spec(1); b = configs.build(s)
rng = np.random.default_rng(0)
f = rng.standard_normal((16,) + b["grid"].counts)
f[2] = 0
for method in ("auto", "block-lu"):
    cache = FactorizationCache(method=method)
    u, _ = diagonal_sweep_solve(torch.from_numpy(f.astype(np.complex128)).cuda(), b["partition"], b["ops"],
                                cache, warn_collar=False)
    uh, _ = diagonal_sweep_solve(torch.from_numpy(f.astype(np.complex128)).pin_memory(), b["partition"],
                                 b["ops"], cache, warn_collar=False)
    assert np.array_equal(u.values.cpu().numpy(), uh.values.numpy())
torch.cuda.synchronize()
print("sanitize run ok")
