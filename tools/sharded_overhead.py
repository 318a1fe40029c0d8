"""Per-application cost of the sharded protocol at world size 1 on one B200
(config 2, 16 RHS): the unsharded plan (CUDA-graph replay) against the
multi-process runner (DistributedShardedSweep, NCCL world 1) with the
device-side flag barrier and with the NCCL-token barrier between launches.
At world size 1 no bytes cross NVLink: the difference is the per-launch
protocol (eager launch issue, one barrier per launch, the final all-reduce).

usage: python tools/sharded_overhead.py [config] [reps]"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2002_05327_b200 import FactorizationCache, configs  # noqa: E402
from paper_2002_05327_b200.ddm import device_plan  # noqa: E402
from paper_2002_05327_b200.sharded import DistributedShardedSweep  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    s = configs.spec(cfg)
    b = configs.build(s)
    part, ops = b["partition"], b["ops"]
    f = configs.sources(s, b["grid"])
    R = f.shape[0]
    fd = torch.from_numpy(f.reshape(R, -1)).cuda()
    cache = FactorizationCache()
    dp = device_plan(part, ops, cache, None, R)
    out = {"config": s.name, "nrhs": R, "unsharded_graph_ms": timed(lambda: dp.apply(fd), reps)}
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29711")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        for bar in ("device", "nccl"):
            sh = DistributedShardedSweep(part, ops, R, cache=cache, barrier=bar)
            out[f"sharded_world1_{bar}_barrier_ms"] = timed(lambda: sh.apply(fd), reps)
            out["launches_per_application"] = sh.plan.nlaunch()
            del sh
    finally:
        dist.destroy_process_group()
    out["t"] = time.strftime("%Y-%m-%dT%H:%M:%S")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
