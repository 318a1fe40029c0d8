"""Command-line drivers (reference `diagsweep/cli.py`, same commands, flags,
artifacts and exit codes) on the batched GPU path.

    python -m paper_2002_05327_b200 solve --config run.ini --out out/
    python -m paper_2002_05327_b200 decay --config run.ini
    python -m paper_2002_05327_b200 precond-study --config run.ini

Flags: --config INI, --out DIR (default "out"), --seed, --threads (host
threads for the host-side assembly), --set SECTION.KEY=VALUE (repeatable).
Exit codes: 0 success, 2 configuration error, 3 non-convergence / solver
error, 4 I/O failure (cli.py:39-41).  Artifacts carry the resolved config's
SHA-256 exactly as the reference writes them (solve_report.json, field.f64le
+ sidecar, quicklook.pgm, residuals.csv, events.jsonl, decay_<NxM>.csv,
decay_report.json, precond_study.csv).

Not provided (outside the hot path): `convergence` (refinement
study against the semi-analytic radial reference, reference.py) and
`pipeline` (the analytic MPI pipeline timing model, pipeline.py); both exit
with code 2 and say so.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
from pathlib import Path

import numpy as np

from . import drivers
from .artifacts import dump_field, write_pgm
from .errors import ConfigurationError, ModelError, SolverError
from .runconfig import load_config

EXIT_CONFIG, EXIT_NOCONV, EXIT_IO = 2, 3, 4


def _csv(path: Path, cfg):
    fh = open(path, "w", newline="")
    fh.write(f"# config sha256: {cfg.sha256}\n")
    return fh


def cmd_solve(cfg, out: Path, rng) -> int:
    events = cfg.getbool("output", "event_log")
    grid, partition, ops, gop = drivers.build_problem(cfg)
    f = cfg.build_source(grid, rng)
    u, info, ddm_rep, kry = drivers.solve_once(cfg, f, partition, ops, gop, events)
    if cfg.getbool("output", "field_dump"):
        dump_field(u, out / "field.f64le")
    if cfg.getbool("output", "quicklook"):
        write_pgm(u, out / "quicklook.pgm")
    if kry is not None and cfg.getbool("output", "residual_csv"):
        kry.write_residual_csv(out / "residuals.csv", f"config sha256: {cfg.sha256}")
    if ddm_rep is not None and events:
        ddm_rep.write_event_log(out / "events.jsonl")
    (out / "solve_report.json").write_text(json.dumps(info, indent=2))
    print(json.dumps(info))
    return EXIT_NOCONV if kry is not None and not kry.converged else 0


def cmd_decay(cfg, out: Path, rng) -> int:
    skip = cfg.getint("decay", "fit_skip")
    floor = cfg.getfloat("decay", "floor")
    report = {"config_sha256": cfg.sha256, "partitions": {}}
    if cfg.get("problem", "source") == "shots":
        report["shots"] = cfg.getpairs("problem", "shots")
    for counts in cfg.decay_partitions():
        name = "x".join(map(str, counts))
        hist = drivers.decay_history(cfg, counts)
        with _csv(out / f"decay_{name}.csv", cfg) as fh:
            w = csv.writer(fh)
            w.writerow(["iteration", "relative_residual"])
            w.writerows([k, f"{h:.6e}"] for k, h in enumerate(hist))
        rate = drivers.fit_decay_rate(hist, skip, floor)
        report["partitions"][name] = {"rate_log10_per_iteration": rate,
                                      "final_residual": float(hist[-1])}
        print(f"partition {name}: decay {rate:.3f} log10/iteration")
    rates = [p["rate_log10_per_iteration"] for p in report["partitions"].values()]
    if len(rates) >= 2:
        report["rate_ratio"] = rates[0] / rates[1]
    (out / "decay_report.json").write_text(json.dumps(report, indent=2))
    return 0


def cmd_precond_study(cfg, out: Path, rng) -> int:
    rows = []
    for cells, counts, freq in drivers.precond_rows(cfg):
        sub, grid, partition, ops, gop, f = drivers.precond_case(cfg, cells, counts, freq)
        _, info, _, _ = drivers.solve_once(sub, f, partition, ops, gop)
        part = "x".join(map(str, counts))
        rows.append((cells, part, freq, info["n_iter"], info["converged"], info["wall_time"]))
        print(f"cells {cells} partition {part} freq {freq}: "
              f"n_iter {info['n_iter']} converged {info['converged']}")
    with _csv(out / "precond_study.csv", cfg) as fh:
        w = csv.writer(fh)
        w.writerow(["cells", "partition", "frequency", "n_iter", "converged", "wall_time"])
        w.writerows(rows)
    return EXIT_NOCONV if any(not r[4] for r in rows) else 0


def _not_here(what):
    def cmd(cfg, out, rng):
        raise ConfigurationError(f"{what} is outside the B200 hot path (SURVEY §8); "
                                 "run it with the reference package")
    return cmd


COMMANDS = {
    "solve": cmd_solve,
    "decay": cmd_decay,
    "precond-study": cmd_precond_study,
    "convergence": _not_here("the convergence study (semi-analytic reference)"),
    "pipeline": _not_here("the pipeline timing model"),
}


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_2002_05327_b200",
                                description="Diagonal sweeping DDM for Helmholtz on B200")
    p.add_argument("command", choices=sorted(COMMANDS))
    p.add_argument("--config", help="INI configuration file")
    p.add_argument("--out", default="out", help="artifact directory")
    p.add_argument("--seed", type=int, default=0, help="PRNG seed")
    p.add_argument("--threads", type=int, default=1, help="host thread cap")
    p.add_argument("--set", dest="overrides", action="append", default=[],
                   metavar="SECTION.KEY=VALUE", help="override one config value (repeatable)")
    return p


def _threads(n: int) -> None:
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=n)
    except ImportError:
        pass


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        sets = {}
        for item in args.overrides:
            if "=" not in item:
                raise ConfigurationError(f"--set needs SECTION.KEY=VALUE, got {item!r}")
            k, v = item.split("=", 1)
            sets[k] = v
        cfg = load_config(args.config, overrides=sets)
        _threads(args.threads)
        out = Path(args.out)
        out.mkdir(parents=True, exist_ok=True)
        return COMMANDS[args.command](cfg, out, np.random.default_rng(args.seed))
    except (ConfigurationError, ModelError) as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except SolverError as exc:
        print(f"solver error: {exc}", file=sys.stderr)
        return EXIT_NOCONV
    except OSError as exc:
        print(f"I/O error: {exc}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
