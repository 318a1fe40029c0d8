"""One config-3-size global operator apply (for ncu of the K1 stencil)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2002_05327_b200 import configs
s = configs.spec(3); b = configs.build(s)
gop = b["gop"]; full = b["partition"].grid.full_window(); counts = b["partition"].grid.counts
x = torch.randn((s.nrhs,) + counts, dtype=torch.complex128, device="cuda")
for _ in range(3):
    y = gop.apply(x, region=full)
torch.cuda.synchronize()
print("ok")
