"""Host logic of the pipelined launch schedule (`_engine.launch_schedule`):
every (sweep, subdomain) visit exactly once, each after all of its routed
sources and after the previous writer of every payload slot it writes, at
most `cap` visits per launch.  CPU only (the tables come from the bit-exact
host metadata: step groups ddm.py:198-203, routing transfer.py:90-97)."""
import numpy as np
import pytest

from paper_2002_05327_b200 import configs
from paper_2002_05327_b200._engine import launch_schedule
from paper_2002_05327_b200.ddm import SweepPlan, source_directions
from paper_2002_05327_b200.partition import steps_per_sweep, sweep_step_of
from paper_2002_05327_b200.transfer import next_usable_sweep


def tables(cfg):
    s = configs.spec(cfg)
    part = configs.build(s)["partition"]
    plan = SweepPlan.default(part.dim).directions
    subs = list(part.subdomains())
    lin = {idx: i for i, idx in enumerate(subs)}
    dirs = source_directions(part.dim)
    counts = part.counts
    order = []
    for w, sd in enumerate(plan):
        for t in range(1, steps_per_sweep(counts) + 1):
            for idx in sorted(x for x in subs if sweep_step_of(x, sd, counts) == t):
                order.append((w, lin[idx]))
    xfer_use = np.full((len(plan), len(subs), len(dirs)), -1, np.int32)
    for w in range(len(plan)):
        for sv, idx in enumerate(subs):
            for k, d in enumerate(dirs):
                tgt = tuple(i + c for i, c in zip(idx, d))
                if not all(1 <= i <= n for i, n in zip(tgt, counts)):
                    continue
                use = next_usable_sweep(d, w + 1, plan)
                xfer_use[w, sv, k] = 0 if use is None else use

    def sub_index(sv, d):
        return lin[tuple(i + c for i, c in zip(subs[sv], d))]

    return len(plan), len(subs), order, xfer_use, dirs, sub_index


@pytest.mark.parametrize("cfg,cap,expect", [(2, 7, 50), (2, 8, 46), (1, 7, None), (4, 10**6, 50)])
def test_launch_schedule_respects_dependencies(cfg, cap, expect):
    nsw, nsub, order, xu, dirs, sub_index = tables(cfg)
    launches = launch_schedule(nsw, nsub, order, xu, dirs, sub_index, None, cap)
    seen = [v for L in launches for v in L]
    assert sorted(seen) == sorted(order) and len(seen) == len(set(seen))
    assert all(1 <= len(L) <= cap for L in launches)
    when = {v: i for i, L in enumerate(launches) for v in L}
    writer = {}
    for (w, s) in order:  # sequential order: sources, then slot writers
        for k, d in enumerate(dirs):
            use = int(xu[w, s, k])
            if use < 1:
                continue
            tgt = (use - 1, sub_index(s, d))
            assert when[(w, s)] < when[tgt]
            key = tgt + (k,)
            if key in writer:
                assert when[writer[key]] < when[(w, s)]
            writer[key] = (w, s)
    if expect is not None:
        assert len(launches) == expect
    # fewer launches than the sweep-by-step order whenever visits can overlap
    assert len(launches) <= len(order)


def test_pooled_schedule_factor_locality():
    """Out-of-core factors (config 5: 64 windows, 10 pool slots): the
    factor-local order keeps every dependency and needs fewer factorizations
    per application than the priority-only order (Belady over both)."""
    from paper_2002_05327_b200._engine import belady_slots

    nsw, nsub, order, xu, dirs, sub_index = tables(5)
    base = launch_schedule(nsw, nsub, order, xu, dirs, sub_index, None, 2)
    loc = launch_schedule(nsw, nsub, order, xu, dirs, sub_index, None, 2, resident=10)
    when = {v: i for i, L in enumerate(loc) for v in L}
    assert sorted(when) == sorted(order)
    for (w, s) in order:
        for k, d in enumerate(dirs):
            use = int(xu[w, s, k])
            if use >= 1:
                assert when[(w, s)] < when[(use - 1, sub_index(s, d))]
    _, _, m_base = belady_slots(base, 10)
    _, _, m_loc = belady_slots(loc, 10)
    assert m_loc < m_base
    assert m_loc <= 360
