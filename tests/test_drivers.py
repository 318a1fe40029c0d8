"""Driver layer on the host: the config loader, the
file artifacts and the CLI's error paths against what the REFERENCE's own
CLI wrote (tests/golden/make_golden_drivers.py).  CPU only; the solves
themselves are compared in tests/test_gpu_drivers.py."""
import csv
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2002_05327_b200 import cli, drivers
from paper_2002_05327_b200.artifacts import dump_field, load_field, write_pgm
from paper_2002_05327_b200.runconfig import load_config

G = Path(__file__).resolve().parent / "golden" / "drivers"
SOLVES = ["solve_gmres", "solve_direct", "solve_global", "solve_layered", "solve_3d"]


def _sets(case):
    return dict(s.split("=", 1) for s in json.loads((G / case / "sets.json").read_text()))


def test_config_resolution_matches_reference():
    rec = json.loads((G / "config.json").read_text())
    cfg = load_config(G / "config_input.ini", environ=rec["environ"], overrides=rec["overrides"])
    assert cfg.values == rec["values"]
    assert cfg.sha256 == rec["sha256"]
    assert cfg.omega == rec["omega"]
    g = cfg.build_grid()
    assert list(g.counts) == rec["grid_counts"]
    assert [list(e) for e in g.extents] == rec["grid_extents"]
    assert list(cfg.partition_counts()) == rec["partition_counts"]
    p = cfg.build_profile()
    assert [p.pml_width_points, p.overlap_d_points, p.sigma_max, p.exponent] == rec["profile"]
    assert cfg.getfloat("solver", "tol") == rec["tol"]
    assert cfg.getbool("output", "quicklook") == rec["quicklook"]


@pytest.mark.parametrize("case", SOLVES + ["decay", "precond"])
def test_config_hash_matches_reference_artifacts(case):
    cfg = load_config(G / case / "input.ini", environ={}, overrides=_sets(case))
    if case == "decay":
        want = json.loads((G / case / "decay_report.json").read_text())["config_sha256"]
    elif case == "precond":
        want = (G / case / "precond_study.csv").read_text().splitlines()[0].split(": ")[1]
    else:
        want = json.loads((G / case / "solve_report.json").read_text())["config_sha256"]
    assert cfg.sha256 == want


def test_config_errors_name_file_and_line(tmp_path):
    ini = tmp_path / "bad.ini"
    ini.write_text("[problem]\ndim = 2\nfrequency = fast\n")
    cfg = load_config(ini, environ={})
    with pytest.raises(Exception) as ei:
        cfg.omega
    assert f"{ini}:3" in str(ei.value)
    with pytest.raises(Exception):
        load_config(tmp_path / "missing.ini", environ={})


@pytest.mark.parametrize("case", SOLVES)
def test_field_artifacts_byte_identical(case, tmp_path):
    """load_field/dump_field round trip and write_pgm reproduce the
    reference's bytes for the reference's own solution."""
    u = load_field(G / case / "field.f64le")
    dump_field(u, tmp_path / "field.f64le")
    assert (tmp_path / "field.f64le").read_bytes() == (G / case / "field.f64le").read_bytes()
    assert (json.loads((tmp_path / "field.f64le.json").read_text())
            == json.loads((G / case / "field.f64le.json").read_text()))
    write_pgm(u, tmp_path / "q.pgm")
    assert (tmp_path / "q.pgm").read_bytes() == (G / case / "quicklook.pgm").read_bytes()


def test_fit_decay_rate_on_reference_histories():
    rep = json.loads((G / "decay" / "decay_report.json").read_text())
    cfg = load_config(G / "decay" / "input.ini", environ={})
    for name, want in rep["partitions"].items():
        with open(G / "decay" / f"decay_{name}.csv") as fh:
            rows = [r for r in csv.reader(ln for ln in fh if not ln.startswith("#"))][1:]
        hist = np.array([float(r[1]) for r in rows])
        rate = drivers.fit_decay_rate(hist, cfg.getint("decay", "fit_skip"),
                                      cfg.getfloat("decay", "floor"))
        # the CSV holds 7 significant digits of the history the rate was fit on
        assert rate == pytest.approx(want["rate_log10_per_iteration"], rel=1e-5)


def test_cli_configuration_errors(tmp_path, capsys):
    case = "solve_badmode"
    argv = ["solve", "--config", str(G / case / "input.ini"), "--out", str(tmp_path)]
    for s in json.loads((G / case / "sets.json").read_text()):
        argv += ["--set", s]
    assert cli.main(argv) == int((G / case / "rc.txt").read_text()) == 2
    assert "unknown solver mode" in capsys.readouterr().err
    assert cli.main(["solve", "--set", "nodot=1", "--out", str(tmp_path)]) == 2
    assert cli.main(["pipeline", "--out", str(tmp_path)]) == 2


def test_cli_without_a_gpu_fails_cleanly(tmp_path, capsys):
    """No CUDA device: a solver error (exit 3) naming the missing device,
    never a CPU fallback."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    rc = cli.main(["solve", "--config", str(G / "solve_gmres" / "input.ini"), "--out", str(tmp_path)])
    assert rc == 3
    assert "no CUDA device" in capsys.readouterr().err
