"""The product's host metadata layer vs the reference (golden fixtures):
partition, windows, owned regions, beta00 supports, PML coefficients,
kappa^2, fingerprints, step groups, routing and psi geometry — bit-exact.
Also: the reference's own golden rule tables (pkg/tests/data) when the
reference tree is present in this container."""

import csv
import hashlib
import itertools
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2002_05327_b200 import configs, content_cuts, emits, solve_cuts
from paper_2002_05327_b200.ddm import SweepPlan, cut_mask_to_set
from paper_2002_05327_b200.partition import sweep_step_of
from paper_2002_05327_b200.transfer import next_usable_sweep, rule_allows, transfer_geometry

GOLD = Path(__file__).resolve().parent / "golden"
REF_DATA = Path("/root/reference/pkg/tests/data")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("k", [1, 2, 3, 4, "5r", 5])
def test_host_metadata_bit_exact(k):
    meta = json.loads((GOLD / f"meta_cfg{k}.json").read_text())
    s = configs.spec(k)
    b = configs.build(s)
    part, ops = b["partition"], b["ops"]
    assert [list(x) for x in part.breaks] == meta["breaks"]
    assert b["omega"] == meta["omega"]
    subs = [tuple(x) for x in meta["subdomains"]]
    assert list(part.subdomains()) == subs
    for i, idx in enumerate(subs):
        w, bx = part.window(idx), part.box(idx)
        assert [list(w.lo), list(w.hi)] == meta["window"][i]
        assert [list(bx.lo), list(bx.hi)] == meta["box"][i]
        assert [[sl.start, sl.stop] for sl in part.owned_slices(idx)] == meta["owned"][i]
        sw, sv = part.beta00_support(idx)
        assert [list(sw.lo), list(sw.hi)] == meta["support"][i]
        assert sha(sv) == meta["beta_sha"][i]
        op = ops[idx]
        assert sha(np.concatenate([*op.alpha_nodes, *op.alpha_faces])) == meta["alpha_sha"][i]
        k2 = op.kappa2 if op.kappa2_kind != "axis" else op.kappa2[1]
        assert sha(np.asarray(k2, dtype=np.float64)) == meta["kappa2_sha"][i]
        assert op.fingerprint == meta["fingerprint"][i]
    gop = b["gop"]
    assert sha(np.concatenate([*gop.alpha_nodes, *gop.alpha_faces])) == meta["gop_alpha_sha"]
    plan = SweepPlan.default(part.dim).directions
    dirs = [d for d in itertools.product((-1, 0, 1), repeat=part.dim) if any(d)]
    for sweep, sd in enumerate(plan, 1):
        groups = {}
        for idx in subs:
            groups.setdefault(sweep_step_of(idx, sd, part.counts), []).append(list(idx))
        assert {str(kk): sorted(v) for kk, v in groups.items()} == meta["steps"][str(sweep)]
        for d in dirs:
            assert next_usable_sweep(d, sweep, plan) == meta["routing"][str(sweep)][" ".join(map(str, d))]
    for idx in subs:
        for d in dirs:
            g = transfer_geometry(part, idx, d)
            want = meta["bands"][" ".join(map(str, idx)) + "|" + " ".join(map(str, d))]
            assert (g is None and want is None) or [list(g.band.lo), list(g.band.hi)] == want


def test_rule_tables_golden():
    tab = np.load(GOLD / "rule_tables.npz")
    for dim in (2, 3):
        for r in tab[f"rule_{dim}d"]:
            s, g, u, a = tuple(r[:dim]), tuple(r[dim:2 * dim]), tuple(r[2 * dim:3 * dim]), r[-1]
            assert rule_allows(s, g, u, dim) == bool(a)


@pytest.mark.skipif(not REF_DATA.exists(), reason="reference tree not present")
@pytest.mark.parametrize("dim", (2, 3))
def test_rule_tables_reference_csv(dim):
    rows = list(csv.DictReader(open(REF_DATA / f"rule_table_{dim}d.csv")))
    assert len(rows) == (128 if dim == 2 else 1664)
    parse = lambda s: tuple(int(x) for x in s.split())
    for row in rows:
        assert rule_allows(parse(row["src_dir"]), parse(row["gen_sweep_dir"]),
                           parse(row["use_sweep_dir"]), dim) == bool(int(row["allowed"]))


def test_cut_bookkeeping_and_device_encoding():
    # pkg/tests/test_ddm.py:63-79 semantics
    own = solve_cuts([], True)
    assert own == frozenset()
    cuts = content_cuts((1, 0), own)
    assert cuts == frozenset({(0, -1)})
    assert content_cuts((0, 1), cuts) == frozenset({(0, -1), (1, -1)})
    assert content_cuts((-1, 0), cuts) == frozenset({(0, 1)})
    assert not emits((-1, 0), cuts)
    assert emits((1, 1), cuts)
    assert solve_cuts([cuts, frozenset({(0, -1)})], False) == frozenset({(0, -1)})
    # device bit encoding (bit 2a + (side > 0)) round-trips
    for dim in (2, 3):
        for mask in range(1 << (2 * dim)):
            cs = cut_mask_to_set(mask, dim)
            back = sum(1 << (2 * a + (s > 0)) for a, s in cs)
            assert back == mask
