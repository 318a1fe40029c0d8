"""Subdomain-sharded sweep (paper_2002_05327_b200/sharded.py) on one device
with virtual ranks: same u as the unsharded sweep (floating-point sums of the
ranks' u in a different order: <= 1e-12 relative), identical counters, and
each rank holding only its own factorizations."""
import numpy as np
import pytest
import torch

from paper_2002_05327_b200 import FactorizationCache, configs, diagonal_sweep_solve
from paper_2002_05327_b200.ddm import SweepPlan, device_plan
from paper_2002_05327_b200.sharded import ShardedSweep, block_owners

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
