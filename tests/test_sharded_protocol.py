"""Host protocol of the multi-process sharded sweep (sharded.run_protocol)
on CPU with gloo, world size 2: stand-in plans record their launch calls;
the protocol must initialise first, run every launch on every rank between
barriers in the same order, finalise, and sum u over the ranks."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2002_05327_b200.sharded import block_owners, run_protocol


class StandInPlan:
    def __init__(self, rank, nl=5):
        self.rank, self.nl, self.calls = rank, nl, []

    def nlaunch(self):
        return self.nl

    def apply_range(self, fmin, umin, nrhs, l0, l1, mode):
        self.calls.append((l0, l1, mode))
        if mode & 1:
            umin.zero_()
        for l in range(l0, l1):  # each rank adds its own contribution per launch
            umin += (self.rank + 1) * (l + 1)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = StandInPlan(rank)
    fmin = torch.zeros(3, 2, dtype=torch.complex128)
    umin = torch.full((3, 2), 7.0, dtype=torch.complex128)
    run_protocol(plan, fmin, umin, 2, dist, device="cpu")
    q.put((rank, plan.calls, umin[0, 0].real.item()))
    dist.destroy_process_group()


def test_protocol_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    expect_calls = [(0, 0, 1)] + [(l, l + 1, 0) for l in range(5)] + [(5, 5, 2)]
    total = sum((r + 1) * (l + 1) for r in range(2) for l in range(5))
    for rank, calls, u00 in res:
        assert calls == expect_calls
        assert u00 == total  # u summed over ranks, initialisation zeroed the stale 7


def _worker_custom_barrier(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = StandInPlan(rank)
    fmin = torch.zeros(3, 2, dtype=torch.complex128)
    umin = torch.zeros((3, 2), dtype=torch.complex128)
    log = []

    def barrier():  # the device barrier's place in the protocol (DeviceBarrier.wait)
        log.append(len(plan.calls))
        dist.barrier()

    run_protocol(plan, fmin, umin, 2, dist, device="cpu", barrier=barrier)
    q.put((rank, log, umin[0, 0].real.item()))
    dist.destroy_process_group()


def test_protocol_world2_custom_barrier():
    """With a device barrier the protocol calls it once after the
    initialisation and once after every launch (never a token all-reduce)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker_custom_barrier, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    total = sum((r + 1) * (l + 1) for r in range(2) for l in range(5))
    for rank, log, u00 in res:
        assert log == [1, 2, 3, 4, 5, 6]
        assert u00 == total


def test_block_owners():
    from paper_2002_05327_b200 import configs

    part = configs.build(configs.spec(2))["partition"]
    own = block_owners(part, 4)
    subs = list(part.subdomains())
    assert sorted(set(own)) == [0, 1, 2, 3]
    assert all(own[i] == (idx[0] - 1) // 2 for i, idx in enumerate(subs))
    with pytest.raises(Exception):
        block_owners(part, 9)
