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
buf = (C.c_longlong * (2 * 1024 * 6))()
fn(buf)
tr = np.frombuffer(buf, dtype=np.int64).reshape(2, 1024, 6)
for rank in range(2):
    t = tr[rank]
    n = int(np.argmax(t[:, 0] == 0)) or 1024
    t = t[:n].astype(np.float64)
    stage = np.median(np.diff(t[:, 0]))
    top_wait = np.median(t[:, 1] - t[:, 0])
    top_comp = np.median(t[:, 2] - t[:, 1])
    top_epi = np.median(t[:, 3] - t[:, 2])
    bot_wait = np.median(t[:, 4] - t[:, 3])
    bot_rest = np.median(t[:, 5] - t[:, 4])
    print(f"rank {rank}: stages {n} median cycles: top wait {top_wait:.0f} compute {top_comp:.0f} "
          f"epilogue {top_epi:.0f} | bottom wait {bot_wait:.0f} compute+epilogue {bot_rest:.0f} | stage {stage:.0f}")
