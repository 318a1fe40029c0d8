"""Pins the CPU oracle (oracle/ds_oracle.py) to the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference package
itself (tests/golden/make_golden.py); here the oracle restatement must
reproduce its index maps and coefficients bit-exactly and its solutions to
round-off.  These tests need no GPU.
"""

import hashlib
import itertools
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import ds_oracle as O
from paper_2002_05327_b200 import configs

GOLD = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_for(k):
    s = configs.spec(k)
    b = configs.build(s)
    return s, b, O.Problem(**configs.oracle_problem(s, b))


@pytest.mark.parametrize("k", [1, 2, 3, 4, "5r", 5])
def test_oracle_metadata_bit_exact(k):
    meta = json.loads((GOLD / f"meta_cfg{k}.json").read_text())
    s, b, prob = oracle_for(k)
    assert [list(x) for x in prob.breaks] == meta["breaks"]
    assert list(prob.counts) == meta["counts"]
    subs = [tuple(x) for x in meta["subdomains"]]
    assert prob.subdomains == subs
    check_ops = subs if k != 5 else subs[:3]  # cfg 5 raster windows are large
    clamp = prob.interior_box()
    for i, idx in enumerate(subs):
        lo, hi = prob.window(idx)
        assert [list(lo), list(hi)] == meta["window"][i]
        blo, bhi = prob.box(idx)
        assert [list(blo), list(bhi)] == meta["box"][i]
        (slo, shi), vals = prob.beta00_support(idx)
        assert [list(slo), list(shi)] == meta["support"][i]
        assert sha(vals) == meta["beta_sha"][i]
        if idx in check_ops:
            op = prob.operator((lo, hi), (blo, bhi), clamp)
            assert sha(np.concatenate([*op.alpha_nodes, *op.alpha_faces])) == meta["alpha_sha"][i]
            k2 = op.kappa2 if op.kappa2_kind != "axis" else op.kappa2[1]
            assert sha(np.asarray(k2, dtype=np.float64)) == meta["kappa2_sha"][i]
            assert hashlib.sha1(op.fingerprint_bytes()).hexdigest() == meta["fingerprint"][i]
    # sweep steps and routing
    plan = O.DEFAULT_2D if prob.dim == 2 else O.DEFAULT_3D
    dirs = O.source_directions(prob.dim)
    for sweep, sd in enumerate(plan, 1):
        groups = {}
        for idx in subs:
            groups.setdefault(O.sweep_step(idx, sd, prob.part_counts), []).append(list(idx))
        assert {str(kk): sorted(v) for kk, v in groups.items()} == meta["steps"][str(sweep)]
        for d in dirs:
            assert O.next_usable(d, sweep, plan) == meta["routing"][str(sweep)][" ".join(map(str, d))]
    # psi band geometry
    for idx in subs[:8]:
        wlo, whi = prob.window(idx)
        zero = np.zeros(tuple(h - l + 1 for l, h in zip(wlo, whi)), dtype=np.complex128)
        ops = {}
        for d in dirs:
            key = " ".join(map(str, idx)) + "|" + " ".join(map(str, d))
            nb = tuple(i + c for i, c in zip(idx, d))
            if meta["bands"][key] is None:
                assert any(not 1 <= x <= n for x, n in zip(nb, prob.part_counts))
                continue
            ops[nb] = prob.operator(prob.window(nb), prob.box(nb), clamp)
            res = O.psi(prob, ops, idx, d, zero, zero)
            assert [list(res[1][0]), list(res[1][1])] == meta["bands"][key]
    # inputs regenerate bit-identically
    assert sha(configs.sources(s, b["grid"])) == meta["source_sha"]
    assert (b["c"] is None and meta["velocity_sha"] is None) or sha(b["c"]) == meta["velocity_sha"]


def test_oracle_rule_tables():
    tab = np.load(GOLD / "rule_tables.npz")
    for dim in (2, 3):
        rows = tab[f"rule_{dim}d"]
        for r in rows:
            s, g, u, a = tuple(r[:dim]), tuple(r[dim:2 * dim]), tuple(r[2 * dim:3 * dim]), r[-1]
            assert O.rule_allows(s, g, u, dim) == bool(a)


def test_oracle_ddm_cfg1_matches_reference():
    g = np.load(GOLD / "ddm_cfg1.npz")
    s, b, prob = oracle_for(1)
    f = configs.sources(s, b["grid"])[0]
    assert sha(f) == str(g["source_sha"])
    u, rep = O.ddm_apply(prob, prob.operators(), O.Cache(), f, record=True)
    assert rel(u, g["u"]) <= 1e-12
    assert [rep["solves"], rep["nonzero_solves"], rep["discarded_sources"]] == list(g["counters"])
    assert rep["events"] == json.loads(str(g["events"]))


def _compact_prob(sigma):
    h, n = 0.01, 141
    return O.Problem(((0.0, h * (n - 1)),) * 2, (n, n), (3, 3), 5, 10, sigma, 2, 25.0, ("const", 1.0))


def test_oracle_compact_and_random_sources():
    g = np.load(GOLD / "ddm_compact.npz")
    prob = _compact_prob(float(g["sigma_max"]))
    ops = prob.operators()
    cache = O.Cache()
    u, rep = O.ddm_apply(prob, ops, cache, g["source"], record=True)
    assert rel(u, g["u"]) <= 1e-12
    assert rep["events"] == json.loads(str(g["events"]))
    rng = np.random.default_rng(2)
    fr = rng.normal(size=prob.counts) + 1j * rng.normal(size=prob.counts)
    assert sha(fr) == str(g["random_sha"])
    ur, _ = O.ddm_apply(prob, ops, cache, fr)
    assert rel(ur, g["u_random"]) <= 1e-12


def test_oracle_additive_against_reference():
    """additive_ddm_solve (ddm.py:294-349): oracle vs the reference's own
    outputs (tests/golden/make_golden_additive.py)."""
    g = np.load(GOLD / "ddm_additive.npz")
    prob = _compact_prob(float(g["sigma_max"]))
    ops = prob.operators()
    cache = O.Cache()
    u, rep = O.additive_apply(prob, ops, cache, g["source"])
    assert rel(u, g["u"]) <= 1e-12
    assert rel(u, g["u_diag"]) <= 1e-12  # the reference's own cross-check (test_ddm.py:132-141)
    assert [rep["solves"], rep["nonzero_solves"], rep["discarded_sources"]] == list(g["counters"])
    fns = {" ".join(map(str, k)): v for k, v in rep["first_nonzero_step"].items()}
    assert fns == json.loads(str(g["first_nonzero_step"]))
    rng = np.random.default_rng(7)
    fr = rng.normal(size=prob.counts) + 1j * rng.normal(size=prob.counts)
    assert sha(fr) == str(g["random_sha"])
    ur, rep_r = O.additive_apply(prob, ops, cache, fr)
    assert rel(ur, g["u_random"]) <= 1e-12
    assert [rep_r["solves"], rep_r["nonzero_solves"], rep_r["discarded_sources"]] == \
        list(g["counters_random"])


def mini_raster():
    return configs.Spec("mini-raster", ((0.0, 2.4), (0.0, 0.8)), (240, 80), 10, 10, (4, 2),
                        None, 3, "gmres", "raster", 3, c_range=(1.5, 3.0), noise=0.15,
                        filt=10.0, src_depth_h=5.0)


def test_oracle_raster_ddm_and_gmres():
    g = np.load(GOLD / "raster_mini.npz")
    s = mini_raster()
    b = configs.build(s)
    prob = O.Problem(**configs.oracle_problem(s, b))
    ops = prob.operators()
    f = configs.sources(s, b["grid"])[0]
    assert sha(f) == str(g["source_sha"]) and sha(b["c"]) == str(g["velocity_sha"])
    cache = O.Cache()
    u, _ = O.ddm_apply(prob, ops, cache, f)
    assert rel(u, g["u_ddm"]) <= 1e-12
    x, rep = O.gmres_ddm(prob, ops, prob.global_operator(), cache, f)
    assert rep["n_iter"] == int(g["n_iter"]) and rep["converged"] == bool(g["converged"])
    assert rel(x, g["x_gmres"]) <= 1e-10
    np.testing.assert_allclose(rep["residuals"], g["residuals"], rtol=1e-8)


def test_oracle_3d_both_plans():
    g = np.load(GOLD / "ddm_3d_mini.npz")
    s = configs.Spec("mini-3d", ((0.0, 1.0),) * 3, (24, 24, 24), 4, 4, (2, 2, 2), 2 * np.pi * 3,
                     1, "direct", "constant", 9, centers=((0.3, 0.55, 0.4),))
    b = configs.build(s)
    prob = O.Problem(**configs.oracle_problem(s, b))
    ops = prob.operators()
    f = configs.sources(s, b["grid"])[0]
    assert sha(f) == str(g["source_sha"])
    cache = O.Cache()
    u, rep = O.ddm_apply(prob, ops, cache, f, record=True)
    assert rel(u, g["u"]) <= 1e-12
    assert rep["events"] == json.loads(str(g["events"]))
    alt = ((1, 1, 1), (-1, 1, 1), (1, -1, 1), (1, 1, -1), (-1, -1, 1), (-1, 1, -1), (1, -1, -1),
           (-1, -1, -1))
    u2, _ = O.ddm_apply(prob, ops, cache, f, directions=alt)
    assert rel(u2, g["u_alt"]) <= 1e-12
