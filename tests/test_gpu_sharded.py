"""Subdomain-sharded sweep (paper_2002_05327_b200/sharded.py) on one device
with virtual ranks: u within 1e-10 of the CPU oracle (and within 1e-12 of the
unsharded sweep: the ranks' u are summed in a different order), identical
counters, and each rank holding only its own factorizations; the device-side
cross-rank barrier (ds_barrier_*) with two ranks on two streams."""
import numpy as np
import pytest
import torch

from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve
from paper_2002_05327_b200.ddm import SweepPlan, device_plan
from oracle import ds_oracle as O
from paper_2002_05327_b200.sharded import DeviceBarrier, ShardedSweep, block_owners

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("cfg,nranks,nrhs", [(1, 2, 2), (1, 4, 2), (2, 2, 4), (2, 8, 2)])
def test_sharded_matches_unsharded(cuda, cfg, nranks, nrhs):
    s = configs.spec(cfg)
    b = configs.build(s)
    part, ops = b["partition"], b["ops"]
    f = configs.sources(s, b["grid"])[:nrhs]
    if f.shape[0] < nrhs:  # pad with seeded random sources
        rng = np.random.default_rng(11)
        extra = rng.normal(size=(nrhs - f.shape[0],) + f.shape[1:]) + 1j * rng.normal(
            size=(nrhs - f.shape[0],) + f.shape[1:])
        f = np.concatenate([f, extra])
    fd = torch.from_numpy(np.ascontiguousarray(f).reshape(nrhs, -1)).cuda()
    cache = FactorizationCache()
    dp = device_plan(part, ops, cache, None, nrhs)
    u_ref, _ = dp.apply(fd)
    ref_ctr = dp.counters(nrhs)
    caches = [FactorizationCache() for _ in range(nranks)]
    sh = ShardedSweep(part, ops, nranks, nrhs, caches=caches)
    u = sh.apply(fd)
    assert rel(u.cpu().numpy(), u_ref.cpu().numpy()) <= 1e-12
    prob = O.Problem(**configs.oracle_problem(s, b))
    oops, oc = prob.operators(), O.Cache()
    for r in range(nrhs):
        want, orep = O.ddm_apply(prob, oops, oc, f[r])
        assert rel(u[r].cpu().numpy().reshape(want.shape), want) <= 1e-10, r
    ctr = sh.counters(nrhs)
    for k in ("nonzero", "discarded", "visit_nonzero", "visit_consumed", "visit_emitted", "visit_cut"):
        assert np.array_equal(ctr[k], ref_ctr[k]), k
    # each rank factorized only its own subdomains' operators
    owner = block_owners(part, nranks)
    for r, c in enumerate(caches):
        own_ops = [ops[idx] for s_, idx in enumerate(part.subdomains()) if owner[s_] == r]
        assert 0 < len(c.factorizations(own_ops)) <= len(own_ops)
    # a second application reuses the zeroed slots
    u2 = sh.apply(fd)
    assert rel(u2.cpu().numpy(), u_ref.cpu().numpy()) <= 1e-12


def test_sharded_sequential_schedule(cuda):
    s = configs.spec(1)
    b = configs.build(s)
    part, ops = b["partition"], b["ops"]
    f = configs.sources(s, b["grid"])[:1]
    u_ref, _ = diagonal_sweep_solve(f, part, ops, FactorizationCache(), warn_collar=False)
    sh = ShardedSweep(part, ops, 2, 1, pipelined=False)
    u = sh.apply(torch.from_numpy(f.reshape(1, -1)).cuda())
    assert rel(u.cpu().numpy().reshape(u_ref.values.shape), u_ref.values) <= 1e-12


def test_distributed_sharded_world1(cuda):
    """The multi-process runner on one rank (NCCL, world size 1): IPC handle
    export, the stream-ordered barriers and the final all-reduce run for real;
    the result equals the unsharded sweep."""
    import os

    import torch.distributed as dist

    from paper_2002_05327_b200.sharded import DistributedShardedSweep

    s = configs.spec(1)
    b = configs.build(s)
    part, ops = b["partition"], b["ops"]
    f = configs.sources(s, b["grid"])[:1]
    fd = torch.from_numpy(f.reshape(1, -1)).cuda()
    u_ref, _ = device_plan(part, ops, FactorizationCache(), None, 1).apply(fd)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29600 + os.getpid() % 300))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        sh = DistributedShardedSweep(part, ops, 1)
        u = sh.apply(fd)
        torch.cuda.synchronize()
        assert rel(u.cpu().numpy(), u_ref.cpu().numpy()) <= 1e-12
    finally:
        dist.destroy_process_group()


def test_sharded_3d_staged_path(cuda):
    """Sharding on the 3D staged solve (K2b + K3g): 2x2x2 subdomains, 2 ranks."""
    s = configs.Spec("mini-3d", ((0.0, 1.0),) * 3, (24, 24, 24), 4, 4, (2, 2, 2), 2 * np.pi * 3,
                     1, "direct", "constant", 9, centers=((0.3, 0.55, 0.4),))
    b = configs.build(s)
    part, ops = b["partition"], b["ops"]
    f = configs.sources(s, b["grid"])[:1]
    fd = torch.from_numpy(f.reshape(1, -1)).cuda()
    u_ref, _ = device_plan(part, ops, FactorizationCache(), None, 1).apply(fd)
    sh = ShardedSweep(part, ops, 2, 1)
    u = sh.apply(fd)
    assert rel(u.cpu().numpy(), u_ref.cpu().numpy()) <= 1e-12


def test_device_barrier_two_ranks_two_streams(cuda):
    """Two barrier ranks on one device, each on its own stream (one
    single-warp kernel each, co-resident): every generation completes on
    both, and work queued after a rank's barrier runs only after the other
    rank's work queued before its own barrier."""
    bars = [DeviceBarrier(2, r) for r in range(2)]
    ptrs = [b.arrive_ptr() for b in bars]
    for b in bars:
        b.set_peers(ptrs)
    streams = [torch.cuda.Stream() for _ in range(2)]
    x = torch.zeros(1 << 20, dtype=torch.float64, device="cuda")
    y = torch.zeros(1, dtype=torch.float64, device="cuda")
    for gen in range(1, 6):
        with torch.cuda.stream(streams[0]):
            x.add_(1.0)          # rank 0's work before the barrier
            bars[0].wait()
        with torch.cuda.stream(streams[1]):
            bars[1].wait()
            y.copy_(x[-1:])      # rank 1 reads rank 0's result after the barrier
        torch.cuda.synchronize()
        assert float(y.item()) == gen
    assert bars[0].generation == bars[1].generation == 5
