"""The product's fast host analyze (C++) against the oracle's independent symbolic phase: bit-exact
on every integer array — small configs directly, the full BASELINE configs
against sha256 digests written by tests/golden/make_symbolic_golden.py (oracle only)."""
import hashlib
import json
import os

import numpy as np
import pytest

import gen
import oracle
import paper_2409_14009_b200 as sp

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = ["post", "parent3", "cc3", "ffirst", "fgroup", "perm_final", "sfirst", "sparent", "rows_ptr", "rows",
        "rel_ptr", "rel_anc", "rel_q0", "rel_off", "relind", "parent_final", "cc_final"]


def compare(prob, cap=0.25, pr=0):
    with sp.Solver.from_problem(prob, device=-1, merge_cap=cap, partition_refinement=pr) as h:
        a = h.spchol_export_symbolic()
        o = oracle.Oracle.from_problem(prob, cap=cap, keep_L=True, pr=pr)
        b = o.symbolic()
        for k in KEYS:
            assert np.array_equal(a[k], b[k]), k
        bl = h.spchol_export_blocks()
        for k in ("blk_ptr", "blk_q", "blk_len", "blk_anc", "blk_relind"):
            assert np.array_equal(bl[k], b[k]), k
        assert h.query("NNZ_L") == o.nnzL
        assert h.query("FLOPS_EXACT") == int(o.flops)
        assert h.query("ADDED") == o.added and h.query("NMERGES") == o.nmerges
        # exact pattern of L (spchol_export_factor_csc) against the oracle's row-merge structure (O2)
        Lp, Li, _, _ = h.spchol_export_factor_csc(values=False)
        oLp, oLi, _ = o.L_csc()
        assert np.array_equal(Lp, oLp) and np.array_equal(Li, oLi)
        return h.query("NSUPER")


@pytest.mark.parametrize("name", ["C1", "T1", "T2", "T3", "S2", "S3", "S4", "S5"])
def test_analyze_small_configs(name):
    compare(gen.make(name))


@pytest.mark.parametrize("name", ["C1", "T1", "T2", "T3", "S2", "S3", "S4", "S5"])
def test_analyze_partition_refinement(name):
    """Partition refinement (reading R14): the product's touched-parts refinement against the oracle's
    whole-partition rebuild (O7b) — bit-exact, including the exact structure of the refined order."""
    compare(gen.make(name), pr=1)


@pytest.mark.parametrize("block", range(0, 3))
def test_analyze_partition_refinement_random(block):
    for trial in range(block * 100, block * 100 + 100):
        compare(gen.random_spd(5000 + trial), pr=1)


@pytest.mark.parametrize("cap", [-1.0, 0.0, 0.05, 0.25, 1.0, 10.0])
def test_analyze_merge_caps(cap):
    compare(gen.make("S5"), cap)
    compare(gen.make("C1"), cap)


@pytest.mark.parametrize("block", range(0, 10))
def test_analyze_random_corpus(block):
    for trial in range(block * 100, block * 100 + 100):
        compare(gen.random_spd(1000 + trial))


def test_analyze_grids_misc():
    for args in [(5, 1, 1, 1, 1), (9, 2, 2, 1, 1), (27, 3, 3, 3, 3), (7, 10, 1, 1, 1), (9, 17, 13, 1, 1),
                 (27, 6, 5, 4, 1), (7, 12, 11, 10, 1), (5, 50, 3, 1, 1)]:
        kind, kx, ky, kz, dof = args
        compare(gen.make_grid(kind, kx, ky, kz, dof))


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_analyze_full_configs_against_golden(name):
    path = os.path.join(HERE, "golden", f"symbolic_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = json.load(open(path))
    p = gen.make(name)
    with sp.Solver.from_problem(p, device=-1) as h:
        a = h.spchol_export_symbolic()
        for k in KEYS:
            assert str(a[k].dtype) == g["dtypes"][k], k
            assert _digest(a[k]) == g["sha256"][k], k
        assert h.query("NNZ_L") == g["nnz_L"] and h.query("NSUPER") == g["nsuper"]
        assert h.query("NFUND") == g["nfund"] and h.query("ADDED") == g["added"]
