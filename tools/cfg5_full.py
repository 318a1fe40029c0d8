"""Config 5 at full size on one B200 (BASELINE.json configs[4]).

3D raster medium on a 128 x 128 x 96 interior (145^2 x 113 nodes, 2.38 M),
PML 8, 4 x 4 x 4 subdomains, 32 near-surface sources, DDM-preconditioned
GMRES to 1e-6 through the public API (`gmres_batched` with `apply_M =
diagonal_sweep_solve`).  The dense block-LU factors of the 64 windows need
638 GB; the default FactorizationCache sees that they exceed HBM and runs the
pooled plan: as many factor slots as fit, each launch's missing factors
recomputed on the device (Belady replacement over the launch schedule).
The reference's own path (SuperLU per window) is infeasible here (SURVEY §7:
~5 h and ~45 GB per window); its checks at full size are:

  phase "residual": every window factored into a pool slot and checked with
      ||A x - b|| / ||b|| <= 1e-10 on 2 random RHS, A applied by the K1 stencil;
  phase "map": linearity and bitwise determinism of the DDM map over the
      first launches of an application (u partial sums and payload state);
  phase "gmres": the timed 32-RHS GMRES-DDM solve: RHS/s, iterations,
      factorizations and the time split (factorization vs sweep kernels).

usage: python tools/cfg5_full.py [phase ...] [--config 5|5r] [--budget-slots N] [--out FILE]
Results are appended as JSON lines to --out (default gpurun_out/cfg5_full.jsonl).
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2002_05327_b200 import (FactorizationCache, configs, diagonal_sweep_solve,  # noqa: E402
                                   gmres_batched)
from paper_2002_05327_b200 import _engine  # noqa: E402
from paper_2002_05327_b200.ddm import SweepPlan, device_plan  # noqa: E402


def emit(out, rec):
    rec["t"] = time.strftime("%Y-%m-%dT%H:%M:%S")
    print(json.dumps(rec), flush=True)
    with open(out, "a") as fh:
        fh.write(json.dumps(rec) + "\n")


def cache_for(args, ops):
    if args.budget_slots:
        per = max(_engine.block_lu_bytes(op.window.shape) for op in ops.values())
        return FactorizationCache(device_budget=args.budget_slots * per + per // 2)
    return FactorizationCache(pool_reserve=args.reserve_gb << 30)


def phase_residual(args, s, b, out):
    ops = [b["ops"][i] for i in b["partition"].subdomains()]
    pool = _engine.FactorPool(ops, 1)
    rng = np.random.default_rng(5005)
    worst, tf = 0.0, []
    for i, op in enumerate(ops):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pool.load(i, 0)
        tf.append(time.perf_counter() - t0)
        rhs = rng.standard_normal((2,) + op.window.shape) + 1j * rng.standard_normal((2,) + op.window.shape)
        x = _engine.fact_solve(pool, i, op.window.shape, torch.from_numpy(rhs).cuda())
        for r in range(2):
            ax = op.apply(x[r])
            res = float(torch.linalg.vector_norm(ax - torch.from_numpy(rhs[r]).cuda())
                        / np.linalg.norm(rhs[r]))
            worst = max(worst, res)
        if i % 8 == 7:
            print(f"  windows {i + 1}/{len(ops)}: worst residual {worst:.2e}, "
                  f"factor {np.mean(tf):.2f} s each", flush=True)
    ba, nb, m, nbytes = pool.info(int(np.argmax([_engine.block_lu_bytes(o.window.shape) for o in ops])))
    emit(out, {"phase": "residual", "config": s.name, "windows": len(ops), "rhs_per_window": 2,
               "worst_relative_residual": worst, "pass": worst <= 1e-10,
               "factor_seconds_mean": float(np.mean(tf)), "factor_seconds_max": float(np.max(tf)),
               "largest_window": {"n_b": nb, "m": m, "factor_bytes": nbytes,
                                  "factor_flop": 8 * nb * m ** 3}})


def phase_factor_rate(args, s, b, out):
    """Factorization throughput: k windows factored one by one vs in one batch."""
    ops = [b["ops"][i] for i in b["partition"].subdomains()]
    k = args.batch
    pool = _engine.FactorPool(ops, k)
    sizes = [8 * max(o.window.shape) * (int(np.prod(o.window.shape)) // max(o.window.shape)) ** 3
             for o in ops]
    pick = list(range(k))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for q, i in enumerate(pick):
        pool.load(i, q)
    t_one = time.perf_counter() - t0
    pick2 = list(range(k, 2 * k))
    t0 = time.perf_counter()
    pool.load_many([(i, q) for q, i in enumerate(pick2)])
    t_batch = time.perf_counter() - t0
    f1 = sum(sizes[i] for i in pick) / t_one / 1e12
    f2 = sum(sizes[i] for i in pick2) / t_batch / 1e12
    emit(out, {"phase": "factor_rate", "config": s.name, "windows": k,
               "one_by_one_s": t_one, "batched_s": t_batch,
               "one_by_one_tflops": f1, "batched_tflops": f2})


def phase_map(args, s, b, out):
    """Linearity and bitwise determinism over the first `--launches` launches
    (two fresh plans, so payload slots start empty; no drain needed)."""
    import gc

    part, ops = b["partition"], b["ops"]
    # dense random fields (every visit nonzero, as for GMRES's Krylov vectors):
    # with compactly supported sources the exact-zero and cut masks differ
    # between f0, f1 and f0 + 2 f1 and the map is only piecewise linear
    rng = np.random.default_rng(5)
    shp = (2,) + tuple(b["grid"].counts)
    f = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
    R = 3
    batch = np.stack([f[0], f[1], f[0] + 2.0 * f[1]])
    cache = cache_for(args, ops)
    slots = cache.pool_slots([ops[i] for i in part.subdomains()])
    if slots is None:
        raise SystemExit("expected a pooled plan")
    n = part.grid.node_count()
    fmin = torch.from_numpy(np.ascontiguousarray(batch.reshape(R, n).T)).cuda()
    snaps, loads = [], 0
    for rep in range(2):
        dp = _engine.DevicePlan(part, ops, cache, SweepPlan.default(3).directions, R, pipelined=True,
                                pool_slots=slots)
        L = min(args.launches, len(dp.launches))
        umin = torch.zeros((n, R), dtype=torch.complex128, device="cuda")
        for l in range(L):
            dp.pool.load_many(dp.pool_loads[l])
            dp.apply_range(fmin, umin, R, l, l + 1, (1 if l == 0 else 0) | 2)
        torch.cuda.synchronize()
        snaps.append(umin.clone())
        loads = dp.pool.state()[2]
        nl = len(dp.launches)
        del dp
        gc.collect()
        torch.cuda.empty_cache()
    u = snaps[0]
    lin = float(torch.linalg.vector_norm(u[:, 2] - (u[:, 0] + 2.0 * u[:, 1]))
                / torch.linalg.vector_norm(u[:, 2]))
    det = bool(torch.equal(snaps[0], snaps[1]))
    emit(out, {"phase": "map", "config": s.name, "launches": L, "of": nl, "pool_slots": slots,
               "factorizations": loads, "linearity_rel": lin, "linearity_pass": lin <= 1e-10,
               "bitwise_deterministic": det, "nonzero_u": float(torch.linalg.vector_norm(u))})


def phase_gmres(args, s, b, out):
    part, ops, gop = b["partition"], b["ops"], b["gop"]
    f = configs.sources(s, b["grid"])
    R = f.shape[0]
    full = part.grid.full_window()
    cache = cache_for(args, ops)
    napp = [0]
    plans = []

    tl = [time.perf_counter()]

    def apply_m(v):
        napp[0] += 1
        u, _ = diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)
        if not plans:
            plans.extend(cache._plans.values())
        torch.cuda.synchronize()
        now = time.perf_counter()
        print(f"  application {napp[0]}: {now - tl[-1]:.1f} s, factorizations so far "
              f"{plans[0].pool.state()[2] if plans else -1}", flush=True)
        tl.append(now)
        return u.values

    fd = torch.from_numpy(f).cuda()
    torch.cuda.synchronize()
    free0, total = torch.cuda.mem_get_info()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, reps = gmres_batched(lambda v: gop.apply(v, region=full), apply_m, fd, tol=1e-6)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev_s = e0.elapsed_time(e1) / 1e3
    dp = plans[0]
    owners, slot_bytes, loads = dp.pool.state()
    # true relative residuals of the returned solution
    r = fd - gop.apply(x, region=full)
    relres = (torch.linalg.vector_norm(r.reshape(R, -1), dim=1)
              / torch.linalg.vector_norm(fd.reshape(R, -1), dim=1)).cpu().numpy()
    emit(out, {"phase": "gmres", "config": s.name, "nrhs": R, "nodes": part.grid.node_count(),
               "rhs_per_s": R / wall, "seconds": wall, "device_seconds": dev_s,
               "applications": napp[0], "n_iter": [rp.n_iter for rp in reps],
               "converged": all(rp.converged for rp in reps),
               "max_true_relres": float(relres.max()),
               "pool_slots": dp.pool.nslots, "slot_bytes": slot_bytes,
               "launches_per_application": len(dp.launches),
               "factorizations_per_application": dp.pool_misses, "factorizations_total": loads,
               "factor_seconds": dp.pool_seconds, "sweep_seconds": wall - dp.pool_seconds,
               "free_bytes_at_start": free0,
               "x_norms": [float(v) for v in torch.linalg.vector_norm(x.reshape(R, -1), dim=1).cpu()]})
    if args.save_x:
        np.save(args.save_x, x.cpu().numpy())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("phases", nargs="*", default=["residual", "map", "gmres"])
    ap.add_argument("--config", default="5")
    ap.add_argument("--budget-slots", type=int, default=0, help="force a pool of N slots")
    ap.add_argument("--reserve-gb", type=int, default=40, help="HBM kept free of factor slots")
    ap.add_argument("--launches", type=int, default=10)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--out", default="gpurun_out/cfg5_full.jsonl")
    ap.add_argument("--save-x", default="")
    args = ap.parse_args()
    cfg = int(args.config) if args.config.isdigit() else args.config
    s = configs.spec(cfg)
    t0 = time.perf_counter()
    b = configs.build(s)
    print(f"{s.name}: grid {b['grid'].counts}, {len(b['ops'])} windows, host assembly "
          f"{time.perf_counter() - t0:.1f} s", flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    torch.cuda.set_device(0)
    for ph in args.phases:
        {"residual": phase_residual, "map": phase_map, "gmres": phase_gmres,
         "factor_rate": phase_factor_rate}[ph](args, s, b, args.out)


if __name__ == "__main__":
    main()
