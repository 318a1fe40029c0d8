"""Per-stage phase timeline of K3 v5 from a DS_SOLVE_TRACE5 build.

Builds a traced copy of the library, runs one warm config-2 application,
and prints, per K3 launch (anti-diagonal step), the median cycles of each
phase seen by thread 0 of cluster rank 0 of the first (visit, chunk):
  fwait  stage top -> factor tile mbarrier complete
  wait   -> exchange mbarrier complete (peers' rows landed), re-armed
  comp   -> own warp's product done
  sync1  -> all warps done (split-K partials in shared memory)
  epi    -> split-K sum, chain update, exchange rows stored
  sync2  -> fence + barrier (then thread 0 issues the multicast)
  tail   -> outputs stored
"""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
lib_path = os.environ.get("TRACE_LIB", "/tmp/libdiagsweep_trace5.so")
env = dict(os.environ, NVCC_APPEND_FLAGS="-DDS_SOLVE_TRACE5 " + os.environ.get("TRACE_FLAGS", ""))
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
lib = N.load_library()
dp.apply(fd)
torch.cuda.synchronize()
lib.ds_debug_solve_trace5_reset()
dp.apply(fd)
torch.cuda.synchronize()
buf = (C.c_longlong * (64 * 16 * 160 * 12))()
cnt = C.c_int(0)
lib.ds_debug_solve_trace5(buf, C.byref(cnt))
tr_all = np.frombuffer(buf, dtype=np.int64).reshape(64, 16, 160, 12).astype(np.float64)
RANK = int(os.environ.get("TRACE_RANK", "0"))
tr = tr_all[:, RANK]
# stamp order within a stage (slot numbers of TRACE5 in ds_solve.cu)
if os.environ.get("DS_K3", "v7") == "v7":  # half-steps: top 0-3, bottom 4-7
    order = [0, 1, 2, 3, 4, 5, 6, 7]
    names = ["T.wait", "T.comp", "T.epi", "T.tail", "B.wait", "B.comp", "B.epi"]
elif tr_all[..., 9].any():  # v5: tile issue (8) and operand issue (9) stamped
    order = [0, 8, 9, 1, 2, 3, 4, 5, 6, 7]
    names = ["tile", "aux", "fwait", "wait", "comp", "sync1", "epi", "sync2", "tail"]
else:  # v6: the producer warp streams tiles; 8 = operands issued
    order = [0, 8, 1, 2, 3, 4, 5, 6, 7]
    names = ["aux", "fwait", "wait", "comp", "sync1", "epi", "sync2", "tail"]
print("launch stages  stage_cyc | " + " ".join(f"{n:>6s}" for n in names))
tot = np.zeros(len(names) + 1)
for L in range(min(cnt.value, 64)):
    t = tr[L]
    n = int(np.argmax(t[:, 0] == 0)) or 160
    if n < 4:
        continue
    t = t[1:n - 1]  # skip prologue-affected first and the last stage
    stage = np.median(np.diff(t[:, 0]))
    ph = [np.median(t[:, order[i + 1]] - t[:, order[i]]) for i in range(len(names))]
    tot[:len(names)] += ph
    tot[-1] += 1
    print(f"{L:6d} {n:6d} {stage:9.0f} | " + " ".join(f"{v:6.0f}" for v in ph))
print("mean over launches         | " + " ".join(f"{v / max(1, tot[-1]):6.0f}" for v in tot[:-1]))

# per-rank view of one launch (the middle one): mean cycles per phase
L = int(os.environ.get("TRACE_LAUNCH", str(max(0, min(cnt.value, 64) // 2))))
print(f"\nlaunch {L}: per rank")
print("rank   stage | " + " ".join(f"{n:>6s}" for n in names))
for rk in range(16):
    t = tr_all[L, rk]
    n = int(np.argmax(t[:, 0] == 0)) or 160
    if n < 4:
        continue
    t = t[1:n - 1]
    stage = np.median(np.diff(t[:, 0]))
    ph = [np.median(t[:, order[i + 1]] - t[:, order[i]]) for i in range(len(names))]
    print(f"{rk:4d} {stage:7.0f} | " + " ".join(f"{v:6.0f}" for v in ph))
