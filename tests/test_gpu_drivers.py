"""The drivers' CLI on the GPU against the REFERENCE's own CLI output
(tests/golden/make_golden_drivers.py): same exit codes, iteration counts,
events and artifacts; fields to relative L2 <= 1e-10 (north star), the
reference's GMRES residual histories to their printed digits, decay
histories to 1e-6 above 1e-12 (below that they are round-off floors), and
the batched drivers equal to one RHS at a time."""
import csv
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2002_05327_b200 import cli, drivers
from paper_2002_05327_b200.artifacts import load_field
from paper_2002_05327_b200.runconfig import load_config

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden" / "drivers"
CMD = {"decay": "decay", "precond": "precond-study", "precond_bad": "precond-study"}


def run_case(case, out):
    argv = [CMD.get(case, "solve"), "--config", str(G / case / "input.ini"), "--out", str(out)]
    for s in json.loads((G / case / "sets.json").read_text()):
        argv += ["--set", s]
    rc = cli.main(argv)
    assert rc == int((G / case / "rc.txt").read_text()), case
    return rc


def _rows(path):
    with open(path) as fh:
        return [r for r in csv.reader(ln for ln in fh if not ln.startswith("#"))][1:]


@pytest.mark.parametrize("case", ["solve_gmres", "solve_direct", "solve_global", "solve_layered",
                                  "solve_3d"])
def test_cli_solve_matches_reference(cuda, case, tmp_path):
    run_case(case, tmp_path)
    want = json.loads((G / case / "solve_report.json").read_text())
    got = json.loads((tmp_path / "solve_report.json").read_text())
    assert got["mode"] == want["mode"] and got["config_sha256"] == want["config_sha256"]
    for k in ("n_iter", "converged"):
        assert got.get(k) == want.get(k), k
    u, ref = load_field(tmp_path / "field.f64le"), load_field(G / case / "field.f64le")
    rel = np.linalg.norm(u.values - ref.values) / np.linalg.norm(ref.values)
    print(f"\n{case}: field rel L2 {rel:.2e}, residual {got['residual']:.3e} "
          f"(reference {want['residual']:.3e})")
    assert rel <= 1e-10
    assert got["residual"] == pytest.approx(want["residual"], rel=1e-3, abs=1e-12)
    if (G / case / "residuals.csv").exists():
        a, b = _rows(tmp_path / "residuals.csv"), _rows(G / case / "residuals.csv")
        assert len(a) == len(b)
        for x, y in zip(a, b):
            assert float(x[1]) == pytest.approx(float(y[1]), rel=1e-5, abs=1e-15)
    if (G / case / "events.jsonl").exists():
        assert ((tmp_path / "events.jsonl").read_text().splitlines()
                == (G / case / "events.jsonl").read_text().splitlines())
    q, qr = (np.frombuffer((p / "quicklook.pgm").read_bytes(), np.uint8).astype(int)
             for p in (tmp_path, G / case))
    assert q.shape == qr.shape and np.abs(q - qr).max() <= 1  # 8-bit rounding of equal fields


def test_cli_decay_matches_reference(cuda, tmp_path):
    run_case("decay", tmp_path)
    want = json.loads((G / "decay" / "decay_report.json").read_text())
    got = json.loads((tmp_path / "decay_report.json").read_text())
    assert got["config_sha256"] == want["config_sha256"]
    assert set(got["partitions"]) == set(want["partitions"])
    for name, w in want["partitions"].items():
        a = np.array([float(r[1]) for r in _rows(tmp_path / f"decay_{name}.csv")])
        b = np.array([float(r[1]) for r in _rows(G / "decay" / f"decay_{name}.csv")])
        assert a.shape == b.shape
        big = b > 1e-12
        np.testing.assert_allclose(a[big], b[big], rtol=2e-6)
        assert np.all(a[~big] < 1e-11)
        assert got["partitions"][name]["rate_log10_per_iteration"] == pytest.approx(
            w["rate_log10_per_iteration"], rel=2e-2)


def test_cli_precond_study_matches_reference(cuda, tmp_path):
    run_case("precond", tmp_path)
    a, b = _rows(tmp_path / "precond_study.csv"), _rows(G / "precond" / "precond_study.csv")
    assert [r[:5] for r in a] == [r[:5] for r in b]  # cells, partition, freq, n_iter, converged
    run_case("precond_bad", tmp_path / "bad")


def test_batched_drivers_equal_single_rhs(cuda):
    """decay_history and solve_once over a 3-source batch equal the
    one-source calls (the batch is the B200 extension of the same API)."""
    cfg = load_config(G / "solve_gmres" / "input.ini", environ={})
    grid, part, ops, gop = drivers.build_problem(cfg)
    srcs = np.stack([cfg.with_values(problem={"center": c}).build_source(grid)
                     for c in ("0.4, 0.55", "0.6, 0.3", "0.25, 0.75")])
    hb = drivers.decay_history(cfg, (3, 2), f=srcs, n_it=5)
    ub, info, _, _ = drivers.solve_once(cfg, srcs, part, ops, gop)
    assert hb.shape == (3, 5) and len(info["n_iter"]) == 3
    for r in range(3):
        h1 = drivers.decay_history(cfg, (3, 2), f=srcs[r], n_it=5)
        np.testing.assert_allclose(hb[r], h1, rtol=1e-12, atol=1e-15)
        u1, i1, _, _ = drivers.solve_once(cfg, srcs[r], part, ops, gop)
        assert i1["n_iter"] == info["n_iter"][r]
        rel = np.linalg.norm(ub.values[r] - u1.values) / np.linalg.norm(u1.values)
        assert rel <= 1e-12
