"""Per-stage phase latencies of K3 from a DS_SOLVE_TRACE build.

Builds a traced copy of the library into /tmp, runs one config-2 application
and prints median cycles per phase: wait (vector + factor), compute (+ K
reduction), epilogue + push.
"""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
lib_path = "/tmp/libdiagsweep_trace.so"
env = dict(os.environ, NVCC_APPEND_FLAGS="-DDS_SOLVE_TRACE")
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
fn = lib.ds_debug_solve_trace
buf = (C.c_longlong * (16 * 1024 * 6))()
fn(buf)
tr = np.frombuffer(buf, dtype=np.int64).reshape(16, 1024, 6)
for rank in range(16):
    tt = tr[rank].astype(np.float64)
    n = int(np.argmax(tt[:, 0] == 0)) or 1024
    if n < 3:
        continue
    tt = tt[:n]
    print(f"rank {rank:2d}: items {n}  median cycles: to-first-panel {np.median(tt[:,1]-tt[:,0]):.0f}  "
          f"panels {np.median(tt[:,2]-tt[:,1]):.0f} (of which waiting {np.median(tt[:,4]):.0f})  "
          f"epilogue {np.median(tt[:,3]-tt[:,2]):.0f}  item {np.median(np.diff(tt[:,0])):.0f}")
