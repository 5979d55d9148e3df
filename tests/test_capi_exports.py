"""The C-ABI library loads on a CPU-only box, exports every symbol include/spchol.h declares, and
its host-side paths (validation, host-only analyze, state errors) behave as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

import gen
import paper_2409_14009_b200 as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "spchol.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spchol_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = sp.lib()
    names = header_functions()
    assert len(names) >= 17
    for nm in names:
        assert hasattr(L, nm), nm
    assert sorted(sp.EXPORTS) == names


def test_default_options():
    o = sp.default_options()
    assert o.merge_cap == 0.25 and o.device == 0 and o.use_graph == 1


def _err(fn):
    with pytest.raises(sp.SpcholError) as ei:
        fn()
    return ei.value.code


def test_validation_errors():
    p = gen.make("T1")
    # non-bijective perm
    bad = p.perm.copy()
    bad[0] = bad[1]
    assert _err(lambda: sp.Solver(p.n, p.colptr, p.rowidx, None, bad, device=-1)) == sp.SPCHOL_ERR_VALIDATION
    # missing diagonal (first entry of column 0 replaced)
    ri = p.rowidx.copy()
    ri[p.colptr[3]] = ri[p.colptr[3] + 1] if p.colptr[4] - p.colptr[3] > 1 else 0
    assert _err(lambda: sp.Solver(p.n, p.colptr, ri, None, p.perm, device=-1)) == sp.SPCHOL_ERR_VALIDATION
    # rows not increasing
    ri = p.rowidx.copy()
    j = next(j for j in range(p.n) if p.colptr[j + 1] - p.colptr[j] >= 3)
    ri[p.colptr[j] + 1], ri[p.colptr[j] + 2] = ri[p.colptr[j] + 2], ri[p.colptr[j] + 1]
    assert _err(lambda: sp.Solver(p.n, p.colptr, ri, None, p.perm, device=-1)) == sp.SPCHOL_ERR_VALIDATION
    # row out of range
    ri = p.rowidx.copy()
    ri[p.colptr[p.n] - 1] = p.n
    assert _err(lambda: sp.Solver(p.n, p.colptr, ri, None, p.perm, device=-1)) == sp.SPCHOL_ERR_VALIDATION
    # negative n
    assert _err(lambda: sp.Solver(-1, np.zeros(1, np.int64), np.zeros(0, np.int32), device=-1)) == sp.SPCHOL_ERR_DIMENSION
    # bad block option
    assert _err(lambda: sp.Solver.from_problem(p, device=-1, block=12)) == sp.SPCHOL_ERR_VALIDATION


def test_host_only_handle_state_errors():
    p = gen.make("T2")
    with sp.Solver.from_problem(p, device=-1) as h:
        assert _err(h.spchol_factor) == sp.SPCHOL_ERR_STATE
        assert _err(lambda: h.spchol_solve(np.ones(p.n))) == sp.SPCHOL_ERR_STATE
        assert _err(lambda: h.spchol_set_values(p.values)) == sp.SPCHOL_ERR_STATE
        assert h.query("N") == p.n and h.query("NNZ_A") == p.nnz
        off, ld, _ = h.spchol_export_panels(values=False)
        sym = h.spchol_export_symbolic()
        m = np.diff(sym["rows_ptr"])
        k = np.diff(sym["sfirst"])
        assert np.all(ld >= m) and np.all(ld % 2 == 0)
        assert np.array_equal(np.diff(off), ld.astype(np.int64) * k)
        assert h.query("PANEL_DOUBLES") == off[-1]


def test_n_zero_and_n_one():
    with sp.Solver(0, np.zeros(1, np.int64), np.zeros(0, np.int32), device=-1) as h:
        assert h.query("NSUPER") == 0 and h.query("NNZ_L") == 0
    with sp.Solver(1, np.array([0, 1], np.int64), np.array([0], np.int32), device=-1) as h:
        assert h.query("NSUPER") == 1 and h.query("NNZ_L") == 1


def test_save_load_analysis_roundtrip(tmp_path):
    """spchol_save_analysis / spchol_load_analysis: the loaded handle carries the
    identical symbolic analysis, plan and layout without re-running analyze."""
    p = gen.make("S5")
    path = tmp_path / "s5.spchol"
    with sp.Solver.from_problem(p, device=-1, merge_cap=0.1) as h:
        h.spchol_save_analysis(path)
        a = h.spchol_export_symbolic()
        ba = h.spchol_export_blocks()
        qa = {k: h.spchol_query(k) for k in sp.Q}
    with sp.Solver.spchol_load_analysis(path, device=-1) as g:
        b = g.spchol_export_symbolic()
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        bb = g.spchol_export_blocks()
        for k in ba:
            assert np.array_equal(ba[k], bb[k]), k
        assert {k: g.spchol_query(k) for k in sp.Q} == qa
    bad = tmp_path / "bad.spchol"
    bad.write_bytes(b"not an analysis")
    assert _err(lambda: sp.Solver.spchol_load_analysis(bad, device=-1)) == sp.SPCHOL_ERR_VALIDATION
    # a file with the right magic but truncated or corrupted contents is rejected before use
    raw = bytearray(path.read_bytes())
    import struct
    n = struct.unpack_from("<q", raw, 16)[0]
    corrupt = [bytes(raw[:len(raw) // 2]),                                  # truncated
               bytes(raw[:-4] + struct.pack("<i", 0x7FFFFFFF)),             # last a_pos out of range
               bytes(raw[:16] + struct.pack("<q", n + 1) + raw[24:]),       # n disagrees with the arrays
               bytes(raw[:-8] + struct.pack("<ii", -5, 0))]                 # negative row position
    for data in corrupt:
        bad.write_bytes(data)
        assert _err(lambda: sp.Solver.spchol_load_analysis(bad, device=-1)) == sp.SPCHOL_ERR_VALIDATION


def test_deterministic_option_plan():
    """deterministic=1 (reading C-7): colour classes add launches; RLB is rejected."""
    p = gen.make("S4")
    with sp.Solver.from_problem(p, device=-1, subtree_streams=1) as h0, \
            sp.Solver.from_problem(p, device=-1, deterministic=1) as h1:
        assert h1.query("LAUNCHES") > h0.query("LAUNCHES")
        assert h1.query("NSUPER") == h0.query("NSUPER")
    assert _err(lambda: sp.Solver.from_problem(p, device=-1, deterministic=1, update_mode=1)) == sp.SPCHOL_ERR_VALIDATION


def test_memory_capped_plan():
    """Memory-capped mode on a host-only handle: the factor's device storage stays under the cap with at
    least two subtree batches; a cap below the resident top fails with DEVICE_OOM; the cap is a
    single-GPU option."""
    p = gen.make("S4")
    with sp.Solver.from_problem(p, device=-1) as h:
        full = h.query("ARENA_BYTES")
        assert h.query("NBATCHES") == 0
    for frac in (0.75, 0.6):
        cap = int(frac * full)
        with sp.Solver.from_problem(p, device=-1, device_mem_cap=cap) as h:
            assert h.query("NBATCHES") >= 2 and h.query("ARENA_BYTES") <= cap
            assert h.query("HOST_BYTES") > 0
    with pytest.raises(sp.SpcholError) as e:
        sp.Solver.from_problem(p, device=-1, device_mem_cap=int(0.1 * full))
    assert e.value.code == sp.SPCHOL_ERR_DEVICE_OOM
    with pytest.raises(sp.SpcholError) as e:
        sp.Solver.from_problem(p, device=-1, device_mem_cap=int(0.6 * full), dist_world=2, dist_rank=0)
    assert e.value.code == sp.SPCHOL_ERR_VALIDATION


def test_dist_init_process_default():
    """spchol_dist_init: later analyze calls with the default dist_world build that rank
    of that world (host-only handles: no communicator is attached); world 1 clears the setting; bad
    arguments are VALIDATION errors."""
    p = gen.make("S4")
    with pytest.raises(sp.SpcholError):
        sp.spchol_dist_init(3, 2, b"\0" * 128)
    try:
        sp.spchol_dist_init(1, 3, b"\1" * 128)
        with sp.Solver.from_problem(p, device=-1) as h:
            owner, _, _ = h.spchol_export_mapping()
            assert owner.max() == 2 and (owner < 0).any()
            assert h.query("NMARKERS") > 0
        with sp.Solver.from_problem(p, device=-1, dist_world=2, dist_rank=0) as h:   # explicit options win
            assert h.spchol_export_mapping()[0].max() == 1
    finally:
        sp.spchol_dist_init(0, 1, None)
    with sp.Solver.from_problem(p, device=-1) as h:
        assert (h.spchol_export_mapping()[0] == 0).all()
