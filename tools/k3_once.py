"""One eager (no CUDA graph) config-N DDM application, for ncu captures of
single kernels: ncu -k regex:k_block_solve5 --launch-skip S --launch-count 1."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200.ddm import SweepPlan, device_plan

s = configs.spec(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
b = configs.build(s)
f = configs.sources(s, b["grid"])
part0 = b["partition"]
# 3D constant media: translation classes share factorizations (bench.py does the same)
cache = FactorizationCache(share_translates=part0.dim == 3 and s.medium == "constant")
dp = device_plan(b["partition"], b["ops"], cache, SweepPlan.default(b["partition"].dim), f.shape[0])
dp.enable_graph(False)
fd = torch.from_numpy(f.reshape(f.shape[0], -1)).cuda()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    dp.apply(fd)
torch.cuda.synchronize()
print("ok")
