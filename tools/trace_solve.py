"""Per-stage phase latencies of K3 (row-split, twisted) from a DS_SOLVE_TRACE
build: builds a traced copy of the library (TRACE_LIB, TRACE_FLAGS), runs one
config-2 application and prints per-rank median cycles per phase.
"""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
lib_path = os.environ.get("TRACE_LIB", "/tmp/libdiagsweep_trace.so")
env = dict(os.environ, NVCC_APPEND_FLAGS=os.environ.get("TRACE_FLAGS", "-DDS_SOLVE_TRACE"))
subprocess.run(["bash", str(ROOT / "paper_2002_05327_b200/csrc/build.sh"), lib_path], check=True, env=env)
os.environ["DIAGSWEEP_B200_LIB"] = lib_path

import numpy as np
import torch

from paper_2002_05327_b200 import FactorizationCache, configs
from paper_2002_05327_b200 import _native as N
from paper_2002_05327_b200.ddm import SweepPlan, device_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
cfg = int(cfg) if cfg.isdigit() else cfg
s = configs.spec(cfg)
b = configs.build(s)
f = configs.sources(s, b["grid"])
cache = FactorizationCache()
dp = device_plan(b["partition"], b["ops"], cache, SweepPlan.default(2), f.shape[0])
fd = torch.from_numpy(f.reshape(f.shape[0], -1)).cuda()
dp.apply(fd)
torch.cuda.synchronize()
lib = N.load_library()
buf = (C.c_longlong * (16 * 1024 * 8))()
lib.ds_debug_solve_trace(buf)
tr = np.frombuffer(buf, dtype=np.int64).reshape(16, 1024, 8)
for rank in range(16):
    tt = tr[rank].astype(np.float64)
    n = int(np.argmax(tt[:, 0] == 0)) or 1024
    if n < 3:
        continue
    tt = tt[:n]
    med = lambda a: float(np.median(a))
    print(f"rank {rank:2d}: stage {med(np.diff(tt[:,0])):.0f} | top: factor-wait {med(tt[:,6]-tt[:,0]):.0f} "
          f"vec-wait {med(tt[:,1]-tt[:,6]):.0f} compute {med(tt[:,2]-tt[:,1]):.0f} epilogue {med(tt[:,3]-tt[:,2]):.0f} "
          f"| bottom: factor-wait {med(tt[:,7]-tt[:,3]):.0f} vec-wait {med(tt[:,4]-tt[:,7]):.0f} "
          f"compute+epi {med(tt[:,5]-tt[:,4]):.0f}")
print("raw rank0 stage10:", tr[0, 10].tolist())
print("raw rank5 stage10:", tr[5, 10].tolist())
print("nonzero ranks:", [r for r in range(16) if tr[r].any()])
