"""Multi-rank host logic on CPU (gloo, world_size 2): RHS sharding, the
gather of shards and max-over-ranks timing used by bench.py --gpus N."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2002_05327_b200.distributed import max_over_ranks, rhs_shard, solve_sharded


def test_rhs_shard_partitions_exactly():
    for R in range(0, 70):
        for world in (1, 2, 3, 8):
            spans = [rhs_shard(R, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == R
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        _worker_body(rank, world, port, q)
    except Exception as exc:  # surface child failures to the test
        import traceback

        q.put((rank, False, -1, repr(exc) + traceback.format_exc()))


def _worker_body(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f = torch.arange(7 * 3, dtype=torch.float64).reshape(7, 3).to(torch.complex128) * (1 + 1j)
        seen = []

        def solve(shard):
            seen.append(shard.shape[0])
            return 2 * shard + rank * 0  # identical map on every rank

        out = solve_sharded(f, solve)
        ok = bool(torch.equal(out, 2 * f))
        mx = max_over_ranks(float(rank + 1))
        q.put((rank, ok, seen[0], mx))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(2)), key=lambda r: r[0])
    for r in res:
        assert r[2] != -1, r[3]
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [True, True]
    assert [r[2] for r in res] == [4, 3]  # 7 RHS over 2 ranks
    assert [r[3] for r in res] == [2.0, 2.0]
