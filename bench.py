#!/usr/bin/env python
"""Benchmark: Helmholtz RHS/s of the diagonal-sweeping DDM (BASELINE.json).

Default workload (`--config 2`, the metric's headline): 2D constant medium,
433^2 nodes, 8x8 subdomains, 16 seeded Gaussian sources, one 4-sweep DDM
application over the 16-RHS batch per step.  Inputs are
generated on the host (NumPy float64, pinned seeds) exactly as the CPU
oracle gets them.

* `value`   RHS/s with the sources resident in HBM (device-timed, CUDA
            events, max over ranks), `N * nrhs / t_step`.
* `e2e`     the same metric through the public API `diagonal_sweep_solve`
            with pinned host buffers: H2D of f and D2H of u inside the
            timed region (plus the per-RHS report read-back).
* `roofline` of the dominant kernel (K3 block substitution), timed live with
            CUDA events bracketing every launch inside the timed region.
* `cpu_baseline` the oracle port on a bounded sample, rank 0 at N=1.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port of the pure-Python reference; the reference itself cannot
travel to the GPU box) on the same config, one RHS per step.

Multi-GPU: RHS-parallel replicas (each rank its own seeded 16-RHS batch,
factorizations replicated, no data-path collective), `scaling: weak`.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2002_05327_b200 import configs  # noqa: E402

L2_BYTES = 126 * 2**20


def peaks():
    p = {}
    try:
        p = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    hbm = p.get("hbm_gbs")
    hbm_src = "measured (MEASURED_PEAKS.json)" if hbm else "fallback (B200_PROFILING.md)"
    fp64 = None
    fp64_src = "nominal B200 FP64 40 TFLOP/s (no measurement found)"
    try:
        q = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())
        fp64 = q["dgemm_tflops"]
        fp64_src = f"measured DGEMM (profiles/fp64_peak.json, {q.get('when', '?')})"
    except Exception:
        pass
    return (hbm or 6650.0), hbm_src, (fp64 or 40.0), fp64_src


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_work(dp, nrhs):
    """Subdomain-solve flops and factor bytes per application,
    every (sweep, subdomain) visit counted (the paper's count):
    * block LU (K3): 16 n_b m^2 flop per RHS; the 2 n_b m^2 complex factor
      entries stream once per RHS chunk (K3 clusters take at most 16 RHS);
    * modal (K3m-T, separable operators): two in-slab transforms per
      direction, 16 n_b m (sum_a n_a) flop per RHS (= 16 n_b m^2 in 2D);
      the transform matrices are L2-resident (n_a^2 entries each).
    Returns (flops, factor_bytes, canonical_flops) where canonical_flops is
    SURVEY's 16 n_b m^2 per RHS whatever the backend."""
    flops = fbytes = canon = 0
    chunks = math.ceil(nrhs / 16)
    for f in dp._keep[1]:
        nb, m = f.n_blocks, f.block_size
        canon += 16 * nb * m * m * nrhs
        if f.backend == "separable":
            flops += 16 * nb * m * (sum(f.shape) - f.shape[f.block_axis]) * nrhs
        else:
            flops += 16 * nb * m * m * nrhs
            fbytes += 2 * nb * m * m * 16 * chunks
    return flops * dp.nsweeps, fbytes * dp.nsweeps, canon * dp.nsweeps


def executed_flops(dp, nrhs):
    """Flop the solve kernels actually run in the last application: the
    modal transforms skip exact-zero RHS columns (and all-zero visits), the
    block-LU K3 skips all-zero visits (whole RHS chunks).  From the device
    counters (visit_nonzero [sweeps][subdomains][R])."""
    import numpy as np

    vnz = dp.counters(nrhs)["visit_nonzero"]
    tot = 0
    for s, f in enumerate(dp._keep[1]):
        nb, m = f.n_blocks, f.block_size
        if f.backend == "separable":
            per = 16 * nb * m * (sum(f.shape) - f.shape[f.block_axis])
            tot += per * int(vnz[:, s, :].sum())
        else:
            per = 16 * nb * m * m
            tot += per * nrhs * int((vnz[:, s, :].sum(-1) > 0).sum())
    return tot


def recurrence_bytes(dp, nrhs):
    """K3m-R (mode-wise recurrences) algorithmic bytes per application: per
    visit and nonzero RHS the transformed block is read and the solution
    written (32 n_b m), plus the mode-wise multipliers / inverse pivots once
    per visit with a nonzero RHS (32 n_b m)."""
    vnz = dp.counters(nrhs)["visit_nonzero"]
    tot = 0
    for s, f in enumerate(dp._keep[1]):
        if f.backend == "separable":
            per = 32 * f.n_blocks * f.block_size
            tot += per * (int(vnz[:, s, :].sum()) + int((vnz[:, s, :].sum(-1) > 0).sum()))
    return tot


def step_kernel_bytes(dp, nrhs):
    """Algorithmic HBM bytes per application of the step kernels (SURVEY
    §8(d)), from the last application's counters and the transfer geometry:
      K6 assemble   16 W per visit and RHS (rhs init) + 32 per copied node
                    (own source in sweep 1, every arriving payload band node);
      K5 accumulate 48 |support| per nonzero visit and RHS;
      K4 transfer   16 |ext| + 48 |band| per emitted, non-discarded source
                    and RHS (the cut / emission rules of ddm.py:82-110)."""
    import numpy as np

    from paper_2002_05327_b200.ddm import cut_mask_to_set, emits

    ctr = dp.counters(nrhs)
    vnz, vcut = ctr["visit_nonzero"], ctr["visit_cut"]
    part = dp.partition
    W = [int(np.prod(part.window(i).shape)) for i in dp.subs]
    own = [int(np.prod(part.owned_window(i).shape)) for i in dp.subs]
    sup = [int(np.prod(part.beta00_window(i).shape)) for i in dp.subs]
    k4 = k5 = k6 = 0
    arrived = 0
    for w in range(dp.nsweeps):
        for s in range(dp.nsub):
            k6 += 16 * W[s] * nrhs + (32 * own[s] * nrhs if w == 0 else 0)
            nz = vnz[w, s]
            k5 += 48 * sup[s] * int(nz.sum())
            for r in np.nonzero(nz)[0]:
                cuts = cut_mask_to_set(int(vcut[w, s, r]), dp.dim)
                for k, d in enumerate(dp.dirs):
                    g = dp.geoms[(s, k)]
                    if g is None or int(dp.xfer_use[w, s, k]) <= 0 or not emits(d, cuts):
                        continue
                    band, ext = int(np.prod(g.band.shape)), int(np.prod(g.ext.shape))
                    k4 += 16 * ext + 48 * band
                    arrived += band
    k6 += 32 * arrived
    return {"assemble": k6, "accumulate": k5, "transfer": k4}


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2002_05327_b200 import FactorizationCache, diagonal_sweep_solve
    from paper_2002_05327_b200.ddm import SweepPlan, device_plan

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    s = configs.spec(args.config)
    b = configs.build(s)
    centers = configs.source_centers(s)
    if world > 1 and rank > 0:  # each replica gets its own seeded batch
        rng = np.random.default_rng(10_000 + rank)
        centers = [tuple(c) for c in rng.uniform(0.05, 0.95, (len(centers), len(centers[0])))]
    f_host = configs.sources(s, b["grid"], centers)
    R = f_host.shape[0]
    part, ops = b["partition"], b["ops"]
    # 3D constant media: share factorizations across translation classes
    # (config 4: 27 classes, 76 GB instead of 203 GB)
    share = part.dim == 3 and s.medium == "constant" and args.factor == "block-lu"
    cache = FactorizationCache(method=args.factor, share_translates=share)

    # ---- factorization (timed separately, amortised)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cache.prepare([ops[i] for i in part.subdomains()])
    e1.record()
    torch.cuda.synchronize()
    factor_ms = e0.elapsed_time(e1)
    factor_wall = time.perf_counter() - t0
    # the library's device path: RHS groups pipelined through the sweeps
    # (ddm._group_count); the per-kernel breakdown below uses one ungrouped
    # plan so that its per-class event times do not overlap
    dp_run = device_plan(part, ops, cache, SweepPlan.default(part.dim), R, grouped=True)
    dp = device_plan(part, ops, cache, SweepPlan.default(part.dim), R)
    cur = [dp_run]
    n = part.grid.node_count()
    f_dev = torch.from_numpy(f_host.reshape(R, n)).to(dev)
    nbytes_f = f_host.nbytes
    gmres_mode = s.mode == "gmres"
    rhs_apps = [0]  # RHS-applications of the DDM map (for the roofline)
    iters = {}
    if gmres_mode:
        from paper_2002_05327_b200 import gmres_batched

        gop = b["gop"]
        full = part.grid.full_window()
        counts = part.grid.counts

        def apply_m(v):
            rhs_apps[0] += v.shape[0]
            uu, _ = cur[0].apply(v.reshape(v.shape[0], -1))
            return uu.reshape(v.shape)

        def step():
            x, reps = gmres_batched(lambda v: gop.apply(v, region=full), apply_m,
                                    f_dev.reshape((R,) + counts), tol=1e-6)
            iters["n_iter"] = [r.n_iter for r in reps]
            iters["converged"] = all(r.converged for r in reps)
            return x
    else:
        def step():
            rhs_apps[0] += R
            u, _ = cur[0].apply(f_dev)
            return u

    # ---- warm-up (untimed)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K applications, inputs resident in HBM (CUDA-graph
    # replay, no per-kernel events; the kernel breakdown is a separate pass)
    clocks = ClockSampler(local_rank)
    clocks.start()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    # L2 flush between timed steps: a 256 MiB zero-fill (twice the 126 MB L2)
    # before every step, outside that step's event pair
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    from paper_2002_05327_b200._engine import launch_count

    launches0 = launch_count()
    rhs_apps[0] = 0
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record()
        step()
        evs[i][1].record()
    launches = launch_count() - launches0  # every kernel of ours in the timed region
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    if os.environ.get("BENCH_DEBUG"):
        print("device step ms:", [round(a.elapsed_time(b), 3) for a, b in evs], file=sys.stderr)
    # ---- kernel breakdown: the same K applications again, eager, with CUDA
    # events around every launch group (not part of `value`)
    ktimes = None
    if args.kernel_events:
        cur[0] = dp
        apps0 = rhs_apps[0]
        step()  # the ungrouped plan's first application (graph / tables)
        dp.set_profiling(True)
        dp.kernel_times(reset=True)
        # the modal transforms count the complex multiply-adds they execute
        # (ds_ctx_work): exact-zero RHS columns and skipped all-zero K-chunks
        # are not in the roofline numerator
        from paper_2002_05327_b200 import _engine
        _engine.set_option("count_work", 1)
        _engine.executed_work(reset=True)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        ktimes = dp.kernel_times(reset=True)
        modal_cmacs = _engine.executed_work(reset=True) / args.steps  # per step
        _engine.set_option("count_work", 0)
        dp.set_profiling(False)
        rhs_apps[0] = apps0
        cur[0] = dp_run
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = world * R / (ms / 1e3)

    # ---- e2e: public API, pinned host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        f_pin = torch.from_numpy(f_host).pin_memory()
        if gmres_mode:
            from paper_2002_05327_b200 import gmres_batched

            def e2e_step():
                x, _ = gmres_batched(lambda v: gop.apply(v, region=full),
                                     lambda v: diagonal_sweep_solve(v, part, ops, cache, warn_collar=False)[0].values,
                                     f_pin.reshape((R,) + counts), tol=1e-6)
                return x
        else:
            def e2e_step():
                uu, _ = diagonal_sweep_solve(f_pin, part, ops, cache, warn_collar=False)
                return uu.values
        # warm-up as the timed loop runs it (the previous result stays alive
        # while the next is produced), so the host allocator has both pinned
        # result buffers before timing
        u_host = None
        for _ in range(max(3, args.warmup)):
            u_host = e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        stamps = []
        for _ in range(args.steps):
            u_host = e2e_step()  # pinned host result (input was a pinned host tensor)
            stamps.append(time.perf_counter())
        assert not u_host.is_cuda
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t1) * 1e3 / args.steps
        if os.environ.get("BENCH_DEBUG"):
            print("e2e step ms:", [round((b - a) * 1e3, 2) for a, b in zip([t1] + stamps, stamps)],
                  file=sys.stderr)
        if world > 1:
            tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        e2e = {"value": world * R / (e2e_ms / 1e3), "unit": "RHS/s",
               "h2d_bytes_per_step": int(nbytes_f), "d2h_bytes_per_step": int(nbytes_f),
               "ms_per_step": e2e_ms,
               "api": ("gmres_batched(gop.apply, diagonal_sweep_solve, pinned host f) -> host x"
                       if gmres_mode else "diagonal_sweep_solve(pinned host f) -> host u")}

    # ---- roofline of the dominant kernel (K3)
    hbm, hbm_src, fp64, fp64_src = peaks()
    flops1, _, canon1 = algorithmic_work(dp, 1)
    apps = rhs_apps[0] / max(1, args.steps)  # RHS-applications per step
    flops = flops1 * apps
    fbytes = algorithmic_work(dp, R)[1] * (apps / R)
    modal = any(f.backend == "separable" for f in dp._keep[1])
    roofline = None
    kernels = None
    if ktimes:
        kernels = {k: {"ms_per_app": v[0] / args.steps, "launches_per_app": v[1] / args.steps}
                   for k, v in ktimes.items()}
        solve_ms = ktimes["block_solve"][0] / args.steps
        # roofline on the flop actually executed (zero RHS columns skipped);
        # SURVEY's canonical count (every visit and RHS) reported beside it
        flops_exec = executed_flops(dp, R) * (apps / R) if not gmres_mode else flops
        flops_nzcols = flops_exec  # every K-chunk of the nonzero (visit, RHS) columns
        if modal and modal_cmacs > 0:
            flops_exec = 8.0 * modal_cmacs  # counted by the kernel itself
        ach = flops_exec / (solve_ms / 1e3) / 1e12
        canon_rate = canon1 * apps / (solve_ms / 1e3) / 1e12
        # DRAM traffic of one K3 launch from the committed ncu --set full capture
        # (profiles/k3_traffic_r01.json), beside that launch's algorithmic bytes
        traffic, traffic_note = None, None
        tpath = ROOT / "profiles" / "k3_traffic_r01.json"
        if tpath.exists() and args.config in (2, "2"):
            tj = json.loads(tpath.read_text())
            traffic = tj["dram_bytes"]
            traffic_note = {"launch": tj["launch"], "algorithmic_factor_bytes": tj["algorithmic_factor_bytes"],
                            "traffic_over_algorithmic": tj["traffic_over_algorithmic"],
                            "duration_us": tj["duration_us"], "source": str(tpath.relative_to(ROOT))}
        if modal:
            tpath = ROOT / "profiles" / f"k3m_traffic_cfg{args.config}.json"
            traffic, traffic_note = None, None
            if tpath.exists():
                tj = json.loads(tpath.read_text())
                traffic = tj["dram_bytes"]
                traffic_note = {k: tj[k] for k in tj if k != "dram_bytes"}
                traffic_note["source"] = str(tpath.relative_to(ROOT))
            roofline = {"bound": "tensor", "pipe": "fp64 tensor (DMMA m8n8k4, 3M complex)",
                        "achieved": ach, "peak": fp64, "unit": "TFLOP/s", "frac": ach / fp64,
                        "traffic": traffic, "traffic_per_launch": traffic_note,
                        "peak_source": fp64_src,
                        "kernel": "k_modal_gemm (K3m-T, in-slab transforms of the modal solve)",
                        "algorithmic_per_app": {"flop_executed": flops_exec,
                                                "flop_nonzero_columns": flops_nzcols,
                                                "flop_all_visits": flops,
                                                "canonical_block_lu_flop": canon1 * apps,
                                                "canonical_rate_tflops": canon_rate,
                                                "note": "achieved = executed flop / K3m-T time; "
                                                        "executed = 8 x the complex multiply-adds the "
                                                        "kernel counts itself (ds_ctx_work: exact-zero "
                                                        "RHS columns, all-zero visits and the all-zero "
                                                        "K-chunks of the forward transforms are skipped "
                                                        "and not counted; the 3M product issues 6 real "
                                                        "flop per multiply-add)"},
                        "share_of_step": solve_ms / ms}
        else:
            roofline = {"bound": "tensor", "pipe": "fp64 tensor (DMMA m8n8k4)", "achieved": ach,
                        "peak": fp64,
                        "unit": "TFLOP/s", "frac": ach / fp64, "traffic": traffic,
                        "traffic_per_launch": traffic_note,
                        "peak_source": fp64_src,
                        "kernel": "k_block_solve (K3)",
                        "algorithmic_per_app": {"flop": flops, "factor_bytes": fbytes},
                        "hbm_view": {"achieved_gbs": fbytes / (solve_ms / 1e3) / 1e9, "peak_gbs": hbm,
                                     "frac": fbytes / (solve_ms / 1e3) / 1e9 / hbm,
                                     "peak_source": hbm_src},
                        "share_of_step": solve_ms / ms}
    # ---- HBM rooflines of the step kernels (K4/K5/K6; SURVEY §8(d) bytes)
    kernel_rooflines = None
    if ktimes:
        kb = step_kernel_bytes(dp, R)  # per application of the R-RHS batch
        if modal:
            kb["modal_recurrence"] = recurrence_bytes(dp, R)
        kernel_rooflines = {}
        for cls, nbytes in kb.items():
            kms = ktimes[cls][0] / args.steps
            gbs = nbytes * (apps / R) / (kms / 1e3) / 1e9 if kms > 0 else None
            kernel_rooflines[cls] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                                     "frac": gbs / hbm if gbs else None,
                                     "algorithmic_bytes_per_app": nbytes, "peak_source": hbm_src}
    # ---- K1 stencil (DiscreteOperator.apply on the global grid, the GMRES
    # operator of configs 3/5) over the bench batch, L2 flushed before each
    # call; 32 B per node and RHS (+8 for a raster kappa^2)
    if ktimes and rank == 0:
        gop_k1 = b["gop"]
        full_k1 = part.grid.full_window()
        vk = f_dev.reshape((R,) + part.grid.counts)
        gop_k1.apply(vk, region=full_k1)
        torch.cuda.synchronize()
        k1ms = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gop_k1.apply(vk, region=full_k1)
            e1.record()
            torch.cuda.synchronize()
            k1ms.append(e0.elapsed_time(e1))
        kms = sorted(k1ms)[len(k1ms) // 2]
        k1_bytes = (32 + (8 if gop_k1.kappa2_kind == "full" else 0)) * n * R
        kernel_rooflines = kernel_rooflines or {}
        kernel_rooflines["stencil_K1"] = {
            "bound": "hbm", "achieved": k1_bytes / (kms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": k1_bytes / (kms / 1e3) / 1e9 / hbm, "algorithmic_bytes_per_call": k1_bytes,
            "ms_per_call": kms, "peak_source": hbm_src,
            "call": f"global operator apply over the {R}-RHS batch ({n} nodes), L2 flushed, median of 5"}
    # ---- parity spot check of the timed output (first RHS vs oracle is in tests)
    res = {
        "metric": "Helmholtz RHS/s (2D 8x8 subdomains)" if args.config == 2 else
        f"Helmholtz RHS/s ({s.name})",
        "gmres": iters or None,
        "value": value, "unit": "RHS/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic (seeded Gaussian sources, SURVEY §8(d))",
        "config": {"workload": s.name, "nrhs_per_gpu": R, "grid": list(part.grid.counts),
                   "subdomains": list(part.counts), "sweeps": len(SweepPlan.default(part.dim).directions),
                   "factor_ms": factor_ms, "factor_wall_s": factor_wall,
                   "factor_bytes": cache.total_bytes, "distinct_factorizations": cache.count,
                   "l2": "flushed before every timed step (256 MiB zero-fill outside the "
                         "per-step CUDA events); factors %.2f GB" % (cache.total_bytes / 1e9),
                   "factor_backend": sorted({f.backend for f in dp._keep[1]}),
                   "parallelism": f"rhs-replicas x{world}",
                   "rhs_groups_per_gpu": getattr(dp_run, "groups", 1)},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "roofline": roofline,
        "kernel_rooflines": kernel_rooflines,
        "kernels": kernels,
    }
    return res


def cpu_sample(s, b, n_rhs, threads):
    """Oracle (port) DDM on n_rhs sources of the same workload."""
    from threadpoolctl import threadpool_limits

    from oracle import ds_oracle as O

    prob = O.Problem(**configs.oracle_problem(s, b))
    oops = prob.operators()
    f = configs.sources(s, b["grid"])
    cache = O.Cache()
    with threadpool_limits(threads):
        t0 = time.perf_counter()
        for idx in prob.subdomains:
            cache.get(oops[idx])
        tf = time.perf_counter() - t0
        gop = prob.global_operator() if s.mode == "gmres" else None

        def one(r):
            if gop is not None:
                O.gmres_ddm(prob, oops, gop, cache, f[r % f.shape[0]])
            else:
                O.ddm_apply(prob, oops, cache, f[r % f.shape[0]])

        one(0)  # warm-up (as the reference arm): first-touch of the factors
        t1 = time.perf_counter()
        for r in range(n_rhs):
            one(r)
        ts = time.perf_counter() - t1
    return tf, ts


def run_reference(args):
    s = configs.spec(args.config)
    b = configs.build(s)
    threads = os.cpu_count() or 1
    from threadpoolctl import threadpool_limits

    from oracle import ds_oracle as O

    prob = O.Problem(**configs.oracle_problem(s, b))
    oops = prob.operators()
    f = configs.sources(s, b["grid"])
    cache = O.Cache()
    with threadpool_limits(threads):
        t0 = time.perf_counter()
        for idx in prob.subdomains:
            cache.get(oops[idx])
        tf = time.perf_counter() - t0
        gop = prob.global_operator() if s.mode == "gmres" else None

        def one(r):
            if gop is not None:
                O.gmres_ddm(prob, oops, gop, cache, f[r % f.shape[0]])
            else:
                O.ddm_apply(prob, oops, cache, f[r % f.shape[0]])

        for w in range(args.warmup):
            one(w)
        t1 = time.perf_counter()
        for k in range(args.steps):
            one(args.warmup + k)
        ts = time.perf_counter() - t1
    value = args.steps / ts
    return {
        "impl": "reference", "metric": "Helmholtz RHS/s (2D 8x8 subdomains)" if args.config == 2
        else f"Helmholtz RHS/s ({s.name})",
        "value": value, "unit": "RHS/s", "n_gpus": args.gpus, "device": "host CPU (rank 0)",
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ts * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic (seeded, SURVEY §8(d))",
        "config": {"workload": s.name,
                   "step": ("one GMRES-DDM solve" if s.mode == "gmres" else "one DDM application")
                   + " for one RHS (the reference API is single-RHS)",
                   "factor_s": tf},
        "cpu_baseline": {"value": value, "unit": "RHS/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} single-RHS applications after {args.warmup} warm-up; "
                                   f"factorization {tf:.2f} s excluded"},
        "e2e": {"value": value, "unit": "RHS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def measure_fp64():
    import torch

    out = {}
    for name, dt, mult in (("dgemm_tflops", torch.float64, 2), ("zgemm_tflops", torch.complex128, 8)):
        nn = 8192 if dt == torch.float64 else 4096
        a = torch.randn(nn, nn, dtype=dt, device="cuda")
        bb = torch.randn(nn, nn, dtype=dt, device="cuda")
        for _ in range(2):
            torch.matmul(a, bb)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, bb)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = mult * nn**3 / (best / 1e3) / 1e12
    out["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    out["how"] = "torch.matmul (cuBLAS) fp64 8192^3 and complex128 4096^3, best of 5, CUDA events"
    out["gpu"] = torch.cuda.get_device_name()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="2")
    ap.add_argument("--factor", default="auto", choices=["auto", "block-lu"],
                    help="factorization method ('block-lu': the block LU for every operator)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-rhs", type=int, default=0,
                    help="CPU baseline sample size (0: the config's whole RHS batch)")
    ap.add_argument("--no-kernel-events", dest="kernel_events", action="store_false")
    ap.add_argument("--measure-fp64", action="store_true")
    args = ap.parse_args()
    args.config = int(args.config) if args.config.isdigit() else args.config
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.measure_fp64:
        print(json.dumps(measure_fp64()))
        return
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)))
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, rank, world, local_rank)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s = configs.spec(args.config)
        b = configs.build(s)
        threads = os.cpu_count() or 1
        # the whole benched batch for direct configs (config 2: 16 RHS, ~6 s
        # on 16 cores), one GMRES solve otherwise
        nsample = (args.cpu_sample_rhs or configs.spec(args.config).nrhs) if s.mode != "gmres" else 1
        tf, ts = cpu_sample(s, b, nsample, threads)
        args.cpu_sample_rhs = nsample
        res["cpu_baseline"] = {"value": args.cpu_sample_rhs / ts, "unit": "RHS/s", "cores": threads,
                               "kind": "port",
                               "sample": f"{args.cpu_sample_rhs} single-RHS "
                                         f"{'GMRES-DDM solves' if s.mode == 'gmres' else 'DDM applications'} "
                                         f"after 1 warm-up, of "
                                         f"{s.name} (oracle port, {threads} BLAS threads); "
                                         f"factorization {tf:.2f} s excluded"}
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
