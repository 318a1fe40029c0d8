#!/usr/bin/env python
"""Golden fixtures for the driver layer (CLI, iterative
decay, preconditioner study, field artifacts), produced by running the
REFERENCE's own CLI and config loader in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_drivers.py

Stores (tests/golden/drivers/):
  config.json    resolved values + sha256 + builder outputs of load_config for
                 an INI file with environment and --set overrides
  solve_*/       `diagsweep solve` artifacts (solve_report.json, field.f64le
                 and sidecar, quicklook.pgm, residuals.csv) for small
                 gmres-ddm / direct-ddm / global-direct problems
  decay/         `diagsweep decay` artifacts (decay_*.csv, decay_report.json)
  precond/       `diagsweep precond-study` artifacts (precond_study.csv)
The INI files used are written next to the artifacts (input.ini).
"""

from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "drivers"
sys.path.insert(0, "/root/reference/pkg/src")

from diagsweep import cli as rcli  # noqa: E402  (the reference)
from diagsweep.config import load_config  # noqa: E402

SMALL = """[problem]
dim = 2
frequency = 4
interior = 0,1; 0,1
medium = constant
speed = 1.0
source = gaussian
center = 0.4, 0.55

[discretization]
interior_cells = 48
pml_points = 6
overlap_points = 3

[partition]
counts = 3,2

[solver]
mode = gmres-ddm
"""

CASES = {
    "solve_gmres": (SMALL, []),
    "solve_direct": (SMALL, ["solver.mode=direct-ddm", "output.event_log=true"]),
    "solve_global": (SMALL, ["solver.mode=global-direct"]),
    "solve_layered": (SMALL + "\n", ["problem.medium=layered", "problem.depths=0.3,0.7",
                                     "problem.speeds=1.0,1.4,1.8", "problem.source=shots",
                                     "problem.shots=0.3,0.6; 0.7,0.2"]),
    "solve_3d": ("""[problem]
dim = 3
frequency = 2
interior = 0,1; 0,1; 0,1
center = 0.4, 0.5, 0.6

[discretization]
interior_cells = 16
pml_points = 4
overlap_points = 2

[partition]
counts = 2,2,2

[solver]
mode = gmres-ddm
""", []),
    "decay": (SMALL + "\n[decay]\npartitions = 3x2; 2x2\niterations = 8\nfit_skip = 1\n", []),
    "precond": (SMALL + "\n[precond]\nrows = 24,2x2,2; 32,2x2,3; 36,3x3,3\n", []),
    "precond_bad": (SMALL + "\n[precond]\nrows = 24,2x2,2; 32,3x3,3\n", []),
    "solve_badmode": (SMALL, ["solver.mode=sweep"]),
}
COMMANDS = {"decay": "decay", "precond": "precond-study", "precond_bad": "precond-study"}


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    # config loader: file < environment < --set
    ini = OUT / "config_input.ini"
    ini.write_text(SMALL + "\n[output]\nquicklook = off\n")
    env = {"DIAGSWEEP_SOLVER_TOL": "1e-8", "DIAGSWEEP_PROBLEM_FREQUENCY": "5",
           "UNRELATED": "x"}
    cfg = load_config(ini, environ=env, overrides={"problem.frequency": "6",
                                                   "partition.counts": "2,2"})
    grid = cfg.build_grid()
    prof = cfg.build_profile()
    rec = {"values": cfg.values, "sha256": cfg.sha256, "environ": env,
           "overrides": {"problem.frequency": "6", "partition.counts": "2,2"},
           "omega": cfg.omega, "grid_counts": list(grid.counts),
           "grid_extents": [list(e) for e in grid.extents],
           "partition_counts": list(cfg.partition_counts()),
           "profile": [prof.pml_width_points, prof.overlap_d_points, prof.sigma_max, prof.exponent],
           "tol": cfg.getfloat("solver", "tol"), "quicklook": cfg.getbool("output", "quicklook")}
    (OUT / "config.json").write_text(json.dumps(rec, indent=1, sort_keys=True))
    for name, (text, sets) in CASES.items():
        d = OUT / name
        d.mkdir()
        (d / "input.ini").write_text(text)
        argv = [COMMANDS.get(name, "solve"), "--config", str(d / "input.ini"), "--out", str(d)]
        for s in sets:
            argv += ["--set", s]
        (d / "sets.json").write_text(json.dumps(sets))
        rc = rcli.main(argv)
        (d / "rc.txt").write_text(str(rc))
        print(name, "rc", rc, sorted(p.name for p in d.iterdir()))


if __name__ == "__main__":
    main()
