"""Parity of the CUDA path (through the C ABI) with the CPU oracle — run on a B200 (-m gpu)."""
import numpy as np
import pytest

import gen
import oracle
import paper_2409_14009_b200 as sp
from helpers import backward_error, logdet_from_diag, lower_panel_mask, panel_index_of_pattern
from test_oracle_pins import grid_logdet

pytestmark = pytest.mark.gpu

SYM_KEYS = ["post", "parent3", "cc3", "ffirst", "fgroup", "perm_final", "sfirst", "sparent", "rows_ptr", "rows",
            "rel_ptr", "rel_anc", "rel_q0", "rel_off", "relind", "parent_final", "cc_final"]
TOL_L = 1e-10      # north_star: max|L_gpu - L_oracle| / max|L| <= 1e-10
TOL_BERR = 1e-12   # north_star: ||Ax-b|| / (||A|| ||x||) <= 1e-12


def run_parity(prob, **opts):
    o = oracle.Oracle.from_problem(prob, pr=opts.get("partition_refinement", 0))
    s_or = o.symbolic()
    assert o.factor() == -1
    Lp, Li, Lx = o.L_csc()
    with sp.Solver.from_problem(prob, **opts) as h:
        s_gpu = h.spchol_export_symbolic()
        for k in SYM_KEYS:                                   # bit-exact symbolic
            assert np.array_equal(s_gpu[k], s_or[k]), k
        assert h.spchol_factor() == (-1, -1)
        off, ld, pan = h.spchol_export_panels()
        idx = panel_index_of_pattern(s_gpu, off, ld, Lp, Li)
        err = np.abs(pan[idx] - Lx).max() / np.abs(Lx).max()
        assert err <= TOL_L, err
        mask = lower_panel_mask(s_gpu, off, ld, len(pan))
        mask[idx] = False                                    # padding = lower panel part outside the pattern
        assert np.all(pan[mask] == 0.0), "padding entries must stay exactly 0"
        cLp, cLi, cLx, npad = h.spchol_export_factor_csc()      # the exact factor in CSC
        assert np.array_equal(cLp, Lp) and np.array_equal(cLi, Li) and npad == 0
        assert np.abs(cLx - Lx).max() <= TOL_L * np.abs(Lx).max()
        xstar, b = gen.rhs(prob)
        x = h.spchol_solve(b)
        assert backward_error(prob, x, b) <= TOL_BERR
        diag = h.spchol_export_diagonal()
        assert np.array_equal(diag, pan[off[:-1][np.repeat(np.arange(len(ld)), np.diff(s_gpu["sfirst"]))]
                                         + (np.arange(prob.n) - np.repeat(s_gpu["sfirst"][:-1], np.diff(s_gpu["sfirst"])))
                                         * (np.repeat(ld, np.diff(s_gpu["sfirst"])).astype(np.int64) + 1)])
    return err


@pytest.mark.parametrize("small", [0, -1, 16])
@pytest.mark.parametrize("name", ["C1", "T1", "T2", "T3", "S2", "S3", "S4", "S5"])
def test_parity_configs(name, small):
    """small = fused small-supernode kernel cutoff (0 default, -1 never: everything tiled)."""
    run_parity(gen.make(name), small_max_k=small)


@pytest.mark.parametrize("vr", [1, 2, 3, 8])
@pytest.mark.parametrize("name", ["C1", "S2", "S4", "S5"])
def test_parity_subtree_streams(name, vr):
    """Single-GPU subtree concurrency (independent subtrees on their own stream pairs)."""
    run_parity(gen.make(name), subtree_streams=vr)
    run_parity(gen.make(name), subtree_streams=vr, small_max_k=-1, use_graph=0)


@pytest.mark.parametrize("block", [8, 16, 24, 40])
def test_parity_block_sizes(block):
    """cdiv block widths that leave ragged block columns (k not a multiple of the block)."""
    run_parity(gen.make("S5"), block=block, small_max_k=-1)
    run_parity(gen.make("T3"), block=block, small_max_k=-1)
    run_parity(gen.make("S4"), block=block)


@pytest.mark.parametrize("trial", range(0, 40))
def test_parity_random_corpus(trial):
    run_parity(gen.random_spd(trial))
    run_parity(gen.random_spd(trial), small_max_k=-1)


def test_parity_no_graph_and_refactor():
    p = gen.make("S4")
    with sp.Solver.from_problem(p, use_graph=0) as h:
        h.spchol_factor()
        d1 = h.spchol_export_diagonal()
        h.spchol_factor()            # refactor with the same values: identical up to RED ordering
        d2 = h.spchol_export_diagonal()
        assert np.abs(d1 - d2).max() <= 1e-12 * np.abs(d1).max()
        ref = grid_logdet(27, (20, 20, 20), 1)
        assert abs(logdet_from_diag(d1) - ref) <= 1e-10 * abs(ref)


@pytest.mark.parametrize("name", ["T3", "S4"])
def test_not_spd_first_failing_column(name):
    p = gen.make(name)
    with sp.Solver.from_problem(p, device=-1) as h0:
        pf = h0.spchol_export_symbolic()["perm_final"]
    for j0 in (0, 5, p.n // 3, p.n - 1):
        i0 = int(np.where(pf == j0)[0][0])
        vals = p.values.copy()
        vals[p.colptr[i0]] = -1.0
        q = gen.Problem(p.name, p.n, p.colptr, p.rowidx, vals, p.perm)
        assert oracle.Oracle.from_problem(q).factor() == j0
        with sp.Solver.from_problem(q, small_max_k=(-1 if j0 % 2 else 0)) as h:
            with pytest.raises(sp.NotSPDError) as ei:
                h.spchol_factor()
            assert ei.value.fail_col == j0 and ei.value.fail_col_orig == i0
            with pytest.raises(sp.SpcholError):
                h.spchol_solve(np.ones(p.n))


def test_edge_cases():
    # n = 1; diagonal A; dense A; forest (block diagonal); arrow
    for D in (np.array([[9.0]]), np.diag(np.arange(1.0, 30.0)),
              np.eye(70) * 80 + np.tril(np.full((70, 70), 1.0), -1),
              np.kron(np.eye(3), np.eye(20) * 4 + np.diag(np.full(19, -1.0), -1))):
        run_parity(gen.from_dense_lower(D))
    n = 50
    D = np.eye(n) * 60
    D[n - 1, :n - 1] = 1.0
    run_parity(gen.from_dense_lower(D))


@pytest.mark.parametrize("name", ["S3", "S4", "S5", "T2"])
def test_parity_tma_tiles(name, monkeypatch):
    """The TMA + mbarrier variant of the tile kernels (SPCHOL_TMA=1): same parity bar."""
    monkeypatch.setenv("SPCHOL_TMA", "1")
    run_parity(gen.make(name), small_max_k=-1)
    run_parity(gen.make(name), block=40, small_max_k=-1)


@pytest.mark.parametrize("name", ["C1", "T2", "T3", "S2", "S3", "S4", "S5"])
def test_parity_rlb(name):
    """RLB: block-pair updates straight into the ancestor panels give the same factor."""
    run_parity(gen.make(name), update_mode=1, small_max_k=-1)
    run_parity(gen.make(name), update_mode=1)


@pytest.mark.parametrize("trial", range(0, 20))
def test_parity_rlb_random(trial):
    run_parity(gen.random_spd(trial), update_mode=1, small_max_k=-1)


def test_load_analysis_then_refactor(tmp_path):
    """A handle rebuilt from a saved analysis factors new values (values-only refactorization)."""
    p = gen.make("S4")
    path = tmp_path / "s4.spchol"
    with sp.Solver.from_problem(p, device=-1) as h0:
        h0.spchol_save_analysis(path)
    vals = p.values * 2.0                        # 2A: L scales by sqrt(2)
    with sp.Solver.spchol_load_analysis(path) as h:
        h.spchol_set_values(vals)
        h.spchol_factor()
        d2 = h.spchol_export_diagonal()
        h.spchol_set_values(p.values)
        h.spchol_factor()
        d1 = h.spchol_export_diagonal()
        assert np.abs(d2 / d1 - np.sqrt(2.0)).max() < 1e-13
        xs, b = gen.rhs(p)
        assert backward_error(p, h.spchol_solve(b), b) <= TOL_BERR


@pytest.mark.parametrize("name", ["S2", "S4", "S5", "T3"])
def test_deterministic_bitwise_reproducible(name):
    """deterministic=1: oracle parity, and the panels are bitwise identical across refactorizations
    and across handles (no FP64 RED in the factor)."""
    p = gen.make(name)
    run_parity(p, deterministic=1)
    run_parity(p, deterministic=1, small_max_k=-1)
    ref = None
    for _ in range(2):
        with sp.Solver.from_problem(p, deterministic=1) as h:
            for _ in range(2):
                assert h.spchol_factor() == (-1, -1)
                _, _, pan = h.spchol_export_panels()
                if ref is None:
                    ref = pan.copy()
                assert np.array_equal(pan.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("trial", range(0, 10))
def test_deterministic_random(trial):
    run_parity(gen.random_spd(300 + trial), deterministic=1)


@pytest.mark.parametrize("name", ["C1", "T2", "T3", "S2"])
@pytest.mark.parametrize("env", [{"SPCHOL_SMALL_WARP": "0"}, {"SPCHOL_SMALL_WARP_MAXM": "128"},
                                 {"SPCHOL_SMALL_WARP_MAXM": "32"}])
def test_parity_small_supernode_paths(name, env, monkeypatch):
    """Small supernodes through each fused path: the CTA-per-supernode kernel only
    (SPCHOL_SMALL_WARP=0), the warp-per-supernode kernel up to m = 128 (4 rows per lane) and up to
    m = 32 (1 row per lane)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    run_parity(gen.make(name))
    run_parity(gen.make(name), deterministic=1)


def run_mock(name, world, env_extra=None, args=(), timeout=1800):
    """Run tests/mock_dist_run.py (every rank a thread on this GPU, NCCL replaced by the blocking
    single-process stand-in tests/mock_nccl) and return its JSON record."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ)
    env.update(env_extra or {})
    here = os.path.dirname(os.path.abspath(__file__))
    assert os.path.exists(os.path.join(here, "mock_nccl", "libmocknccl.so")), "build it with make"
    p = subprocess.run([sys.executable, os.path.join(here, "mock_dist_run.py"), name, str(world), *map(str, args)],
                       env=env, capture_output=True, text=True, timeout=timeout)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert lines, p.stdout[-2000:] + p.stderr[-2000:]
    return json.loads(lines[-1])


@pytest.mark.parametrize("name,world,minflops,outer", [
    ("S4", 2, None, None), ("S5", 3, None, None), ("C1", 2, None, None), ("S2", 4, None, None), ("T3", 2, None, None),
    ("S4", 8, None, None),
    # distributed top supernodes (block-column cyclic cdiv, broadcasts, K-split partial U_J)
    ("S4", 2, "0", None), ("S4", 4, "0", "1"), ("S5", 3, "0", "1"), ("S2", 4, "0", "1"), ("T3", 2, "0", "1"),
    ("S4", 8, "0", "1"), ("S5", 8, "0", None), ("S3", 5, "0", "1"), ("S2", 8, "0", "1")])
def test_distributed_nccl_path_mock(name, world, minflops, outer):
    """The multi-GPU factor and solve through the library's real NCCL code path (communicator
    splits per top rank group, grouped send/recv of the update runs + extend-add, block-column
    broadcasts, the solve's per-block reduces / broadcasts and final all-reduce), each rank a thread
    on this GPU with its own per-rank arena: no hang (same call order on every rank), the sum of the
    ranks' panel exports matches the oracle with every padding entry exactly 0, backward error
    within the bound, every rank returns the same solution, two factor + solve rounds."""
    env = {}
    if minflops is not None:
        env["SPCHOL_DIST_MINFLOPS"] = minflops
    if outer is not None:
        env["SPCHOL_OUTER"] = outer
    r = run_mock(name, world, env)
    assert r["ok"], r
    assert r["lerr"] <= TOL_L and r["berr"] <= TOL_BERR and r["ranks_agree"], r
    assert r["padding_nonzeros"] == 0, r
    if minflops == "0" and name not in ("T3",):
        assert r["ntop_dist"] > 0


@pytest.mark.parametrize("name,world", [("S4", 3), ("S5", 2)])
def test_distributed_partition_refinement_mock(name, world):
    """The multi-GPU path on a partition-refined analysis (reading R14): same parity bar as above."""
    r = run_mock(name, world, {"MOCK_PR": "1", "SPCHOL_DIST_MINFLOPS": "0"})
    assert r["ok"], r
    assert r["lerr"] <= TOL_L and r["berr"] <= TOL_BERR and r["ranks_agree"] and r["padding_nonzeros"] == 0, r


@pytest.mark.parametrize("name,world", [("C4", 2), ("C4", 4), ("C4", 8), ("C5", 2), ("C5", 4)])
def test_distributed_fullsize_mock(name, world):
    """The north_star's multi-GPU configs (C4 at 2/4/8 ranks, C5 at 2/4) through the real NCCL code
    path on one GPU (ranks as threads, per-rank arenas): log det of the grid operator from its
    closed-form eigenvalues (the whole diagonal of L), backward error, all ranks agree, and the
    exact-result check (L L^T)(i, j) = C_f(i, j) on sampled columns of the top three levels — the
    distributed supernodes — with the panels summed over the ranks' exports."""
    r = run_mock(name, world, {"MOCK_FULL": "1"}, timeout=3600)
    assert r["ok"], r
    assert r["logdet_rel_err"] <= 1e-10, r
    assert r["berr"] <= TOL_BERR and r["ranks_agree"], r
    assert r["llt_err"] <= 1e-12 and r["llt_entries"] >= 10 ** 5, r
    assert r["ntop_dist"] > 0
    print(name, world, {k: r[k] for k in ("factor_s", "arena_bytes", "send_bytes", "recv_bytes", "llt_err")})


@pytest.mark.parametrize("name", ["S3", "S4", "S5"])
@pytest.mark.parametrize("env", [{"SPCHOL_LEFT_INNER": "1"}, {"SPCHOL_NO_NEXT_SPLIT": "1"}, {"SPCHOL_REST_SMEM": "60000"},
                                 {"SPCHOL_PDL": "0"}, {"SPCHOL_POTRF9": "1", "SPCHOL_PANEL": "0"}, {"SPCHOL_PANEL": "0"}])
def test_parity_schedule_options(name, env, monkeypatch):
    """Scheduling variants of the large-supernode cdiv (left-looking in-block updates, NEXT as one
    launch, capped trailing-stream residency, no programmatic dependent launch, the right-looking
    potrf9 reference kernel, no fused outer-block path): same factor, same solve."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    run_parity(gen.make(name), small_max_k=-1)
    run_parity(gen.make(name), small_max_k=-1, block=64)


def test_device_footprint_query():
    """SPCHOL_Q_DEVICE_BYTES: the handle's device memory covers the panel arena, the kept diagonal
    inverses and the plan; a host-only handle owns none."""
    prob = gen.make("S4")
    with sp.Solver.from_problem(prob) as h:
        nb = h.query("DEVICE_BYTES")
        assert nb >= 8 * h.query("PANEL_DOUBLES") + 8 * h.query("NNZ_A")
        assert nb < 64 * (h.query("PANEL_DOUBLES") + h.query("NNZ_A")) + (64 << 20)
    with sp.Solver.from_problem(prob, device=-1) as h:
        assert h.query("DEVICE_BYTES") == 0


@pytest.mark.parametrize("name,world,frac,minflops", [("S4", 2, 0.1, "0"), ("S4", 4, 0.97, "0"), ("S5", 3, 0.5, None)])
def test_distributed_not_spd_mock(name, world, frac, minflops):
    """A failing pivot on one rank (in a subtree or in a distributed top supernode): every rank
    reports the sequential first failing column (all-reduce(min) of the fail flags) through the
    real NCCL code path over the single-process stand-in."""
    r = run_mock(name, world, {"SPCHOL_DIST_MINFLOPS": minflops} if minflops is not None else {}, args=(frac,))
    assert r["ok"], r


def _arena(prob):
    with sp.Solver.from_problem(prob, device=-1) as h:
        return h.query("ARENA_BYTES")


@pytest.mark.parametrize("name,frac", [("S2", 0.6), ("S3", 0.6), ("S4", 0.6), ("S5", 0.6), ("C1", 0.6), ("T3", 0.75)])
def test_memory_capped_parity(name, frac):
    """Memory-capped mode (f-4): the device storage is capped below the panel footprint; the
    subtree batches run in one device window and go to pinned host memory, the solve streams them
    back.  Same parity bar as the resident factor (oracle, padding, exact-pattern CSC, solve)."""
    prob = gen.make(name)
    cap = int(frac * _arena(prob))
    run_parity(prob, device_mem_cap=cap)
    with sp.Solver.from_problem(prob, device_mem_cap=cap) as h:
        assert h.query("NBATCHES") >= 2
        assert h.query("ARENA_BYTES") <= cap


def test_memory_capped_fullsize_C3():
    """C3 (n = 262144) with the factor's device storage capped at half its footprint: closed-form log
    det, backward error, and the exact-result check L L^T = C_f on the top levels."""
    from helpers import llt_sample_error, top_level_columns
    p = gen.make("C3")
    cap = int(0.5 * _arena(p))
    with sp.Solver.from_problem(p, device_mem_cap=cap) as h:
        assert h.query("NBATCHES") >= 2 and h.query("ARENA_BYTES") <= cap
        h.spchol_factor()
        h.spchol_factor()
        ld = logdet_from_diag(h.spchol_export_diagonal())
        ref = grid_logdet(p.kind, p.grid, p.dof)
        assert abs(ld - ref) <= 1e-10 * abs(ref)
        xs, b = gen.rhs(p)
        x = h.spchol_solve(b)
        assert backward_error(p, x, b) <= TOL_BERR
        sym = h.spchol_export_symbolic()
        off, ldv, pan = h.spchol_export_panels()
    err, cnt = llt_sample_error(p, sym, off, ldv, pan, top_level_columns(sym, nlev=3, per_sn=3))
    assert err <= 1e-12 and cnt >= 10 ** 4


@pytest.mark.parametrize("name", ["S4", "S5", "C1", "T2"])
@pytest.mark.parametrize("nrhs", [1, 3, 16])
@pytest.mark.parametrize("capped", [False, True])
def test_multi_rhs_solve(name, nrhs, capped):
    """f-1, multiple right-hand sides: nrhs columns with leading dimension ld > n, solved in
    blocks of 4 / 2 / 1 (one pass over L per block), in place (b aliasing x) and out of place; every
    column against the oracle's scalar solve and within the backward-error bound.  Resident and
    memory-capped factor."""
    import ctypes
    prob = gen.make(name)
    o = oracle.Oracle.from_problem(prob)
    assert o.factor() == -1
    n, ld = prob.n, prob.n + 5
    rng = np.random.default_rng(nrhs)
    B = np.zeros((nrhs, ld))                       # column r at B[r, :n] (column-major, ld)
    B[:, :n] = rng.uniform(-1, 1, (nrhs, n))
    opts = {}
    if capped and name == "T2":
        pytest.skip("T2's resident top alone is above any cap below its footprint")
    if capped:
        with sp.Solver.from_problem(prob, device=-1) as h0:
            opts["device_mem_cap"] = int(0.6 * h0.query("ARENA_BYTES"))
    with sp.Solver.from_problem(prob, **opts) as h:
        assert h.spchol_factor() == (-1, -1)
        X = np.full_like(B, 7.0)
        assert h._L.spchol_solve(h._h, sp._vp(B), sp._vp(X), nrhs, ld) == 0
        Y = B.copy()
        assert h._L.spchol_solve(h._h, sp._vp(Y), sp._vp(Y), nrhs, ld) == 0       # aliased b == x
        for r in range(nrhs):
            xr = o.solve(B[r, :n])
            assert np.abs(X[r, :n] - xr).max() <= 1e-10 * np.abs(xr).max()
            assert np.abs(X[r, :n] - Y[r, :n]).max() <= 1e-12 * np.abs(xr).max()   # FP64 RED: rounding order varies
            assert backward_error(prob, X[r, :n], B[r, :n]) <= TOL_BERR
        assert np.all(X[:, n:] == 7.0)             # the padding rows of the ld are untouched


@pytest.mark.parametrize("name", ["S2", "S3", "S4", "S5", "T2"])
@pytest.mark.parametrize("mode", [0, 1])
def test_parity_partition_refinement(name, mode):
    """Partition refinement (f-2, reading R14) with RL (mode 0) and RLB (mode 1):
    bit-exact symbolic arrays against the oracle's O7b, the factor of the refined order within the
    parity bar, padding exactly 0, solve within the backward-error bound."""
    run_parity(gen.make(name), partition_refinement=1, update_mode=mode)


FUSED_ALL = {"SPCHOL_PANEL_MAX_SN": "1000000", "SPCHOL_PANEL_MAX_ROWS": "1000000000"}


def _dense_spd(n, seed, extra_rows=0):
    """Dense SPD block of n columns (one supernode) plus, with extra_rows, a second dense block
    coupled to it, so the first supernode has rows below its diagonal block (m > k)."""
    rng = np.random.default_rng(seed)
    N = n + extra_rows
    D = np.tril(-rng.uniform(0.0, 1.0, (N, N)) / N, -1)
    np.fill_diagonal(D, 2.0 + rng.uniform(0.0, 0.1, N))
    return gen.from_dense_lower(D)


@pytest.mark.parametrize("env", [{}, {"SPCHOL_PDL": "0"}, {"SPCHOL_PANEL_GRID": "3"}])
@pytest.mark.parametrize("name", ["C1", "T3", "S3", "S4", "S5"])
def test_parity_fused_panel_all_levels(name, env, monkeypatch):
    """The fused outer-block cdiv (panel_diag_kernel + panel_below_kernel, lookahead update folded in)
    forced on every level and outer block: same factor, same solve; also without programmatic
    dependent launch (the below launch then runs after the diagonal one) and with a 3-CTA below
    launch (every CTA works through many tasks in ticket order)."""
    for k, v in {**FUSED_ALL, **env}.items():
        monkeypatch.setenv(k, v)
    run_parity(gen.make(name), small_max_k=-1)
    run_parity(gen.make(name))


@pytest.mark.parametrize("n,extra", [(64, 0), (200, 0), (256, 0), (300, 0), (700, 0), (520, 130), (1000, 333)])
def test_parity_fused_panel_dense(n, extra, monkeypatch):
    """Dense blocks held as one or two supernodes: outer blocks of 1-4 inner blocks, a partial last
    block (k mod 64 != 0), rows below the diagonal region and tiles cut by m; fused path vs oracle."""
    for k, v in FUSED_ALL.items():
        monkeypatch.setenv(k, v)
    run_parity(_dense_spd(n, n + extra, extra), small_max_k=-1)


def test_parity_fused_panel_kernel_timing(monkeypatch):
    """Kernel timing serializes every launch on one stream (no PDL): the fused path still completes
    and the per-kind statistics account for its launches."""
    for k, v in FUSED_ALL.items():
        monkeypatch.setenv(k, v)
    p = gen.make("S5")
    o = oracle.Oracle.from_problem(p)
    assert o.factor() == -1
    Lp, Li, Lx = o.L_csc()
    with sp.Solver.from_problem(p, small_max_k=-1) as h:
        h.spchol_enable_kernel_timing(True)
        assert h.spchol_factor() == (-1, -1)
        st = h.spchol_kernel_stats("panel")
        assert st["launches"] > 0 and st["flops"] > 0
        h.spchol_enable_kernel_timing(False)
        cLp, cLi, cLx, _ = h.spchol_export_factor_csc()
        assert np.abs(cLx - Lx).max() <= TOL_L * np.abs(Lx).max()


@pytest.mark.parametrize("name", ["T3", "S4"])
def test_not_spd_fused_panel(name, monkeypatch):
    """A failing pivot inside the fused path is reported as the sequential first failing column."""
    for k, v in FUSED_ALL.items():
        monkeypatch.setenv(k, v)
    test_not_spd_first_failing_column(name)


@pytest.mark.parametrize("name,world,minflops,outer", [("S4", 2, None, None), ("S5", 3, "0", None), ("S4", 4, "0", "1"),
                                                       ("T3", 2, "0", "2")])
def test_distributed_fused_panel_mock(name, world, minflops, outer):
    """The fused outer-block cdiv on every level of the multi-GPU path (own subtrees, undistributed
    top supernodes with the lookahead folded in, distributed top supernodes with their NEXT on the
    next block column's owner), through the real NCCL code path over the single-process stand-in."""
    env = dict(FUSED_ALL)
    if minflops is not None:
        env["SPCHOL_DIST_MINFLOPS"] = minflops
    if outer is not None:
        env["SPCHOL_OUTER"] = outer
    r = run_mock(name, world, env)
    assert r["ok"], r
    assert r["lerr"] <= TOL_L and r["berr"] <= TOL_BERR and r["ranks_agree"], r
    assert r["padding_nonzeros"] == 0, r


@pytest.mark.parametrize("use_graph", [1, 0])
def test_set_values_prezeroed_arena(use_graph):
    """spchol_set_values zeroes the panel arena on a side stream during the upload, and the next factor
    skips its memset (variant graph): factor after set_values, factor again without it (full graph),
    and a refactor with new values all give the oracle's factor; a pending solve is not disturbed by
    the next set_values' zeroing (it waits for the handle's earlier work)."""
    p = gen.make("S4")
    o = oracle.Oracle.from_problem(p)
    assert o.factor() == -1
    _, _, Lx = o.L_csc()
    q = gen.Problem(p.name, p.n, p.colptr, p.rowidx, 4.0 * p.values, p.perm)   # L(4A) = 2 L(A)
    with sp.Solver.from_problem(p, use_graph=use_graph) as h:
        for _ in range(2):
            assert h.spchol_factor() == (-1, -1)
            _, _, cLx, _ = h.spchol_export_factor_csc()
            assert np.abs(cLx - Lx).max() <= TOL_L * np.abs(Lx).max()
        xs, b = gen.rhs(p)
        x = h.spchol_solve(b)
        assert backward_error(p, x, b) <= TOL_BERR
        h.spchol_set_values(q.values)
        assert h.spchol_factor() == (-1, -1)
        _, _, cLx, _ = h.spchol_export_factor_csc()
        assert np.abs(cLx - 2.0 * Lx).max() <= 2.0 * TOL_L * np.abs(Lx).max()
        h.spchol_set_values(p.values)
        assert h.spchol_factor() == (-1, -1)
        _, _, cLx, _ = h.spchol_export_factor_csc()
        assert np.abs(cLx - Lx).max() <= TOL_L * np.abs(Lx).max()
