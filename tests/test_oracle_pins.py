"""Pins of the CPU oracle against things other than itself (CPU only, ``-m "not gpu"``).

Each test names what fixes the expected value: a value the paper prints (tests/golden/fig1.json,
with citations), a closed form, a textbook/library routine (LAPACK via numpy), brute force on
tiny inputs, or an invariant the paper states.
"""
import json
import math
import os

import numpy as np
import pytest

import gen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
FIG1 = json.load(open(os.path.join(HERE, "golden", "fig1.json")))


def fig1_problem():
    D = np.zeros((15, 15))
    for j, rows in FIG1["columns"].items():
        j = int(j)
        for i in rows:
            D[i - 1, j - 1] = FIG1["values"]["diag"] if i == j else FIG1["values"]["off"]
    return gen.from_dense_lower(D, name="fig1")


def dense_of(L_csc, n):
    Lp, Li, Lx = L_csc
    L = np.zeros((n, n))
    for j in range(n):
        L[Li[Lp[j]:Lp[j + 1]], j] = Lx[Lp[j]:Lp[j + 1]] if Lx is not None else 1.0
    return L


def permuted_dense(prob, pf):
    C = np.zeros((prob.n, prob.n))
    C[np.ix_(pf, pf)] = gen.to_dense(prob)
    return C


# ---------------------------------------------------------------- Fig. 1 (paper-printed values)
def test_fig1_etree_and_maximal_partition():
    p = fig1_problem()
    o = oracle.Oracle.from_problem(p, cap=-1, rule=1)
    s = o.symbolic()
    post = s["post"]  # post[new] = paper label - 1
    # etree: parent in paper labels
    par = np.zeros(15, int)
    for new in range(15):
        pn = s["parent3"][new]
        par[post[new]] = 0 if pn < 0 else post[pn] + 1
    assert par.tolist() == FIG1["etree_parent_1based"]["value"]
    # maximal supernodes = Fig. 1's J1..J6
    sets = []
    for J in range(o.nsuper):
        cols = [int(np.where(s["perm_final"] == c)[0][0]) + 1 for c in range(s["sfirst"][J], s["sfirst"][J + 1])]
        sets.append(sorted(cols))
    assert sorted(sets) == sorted(FIG1["supernodes_maximal"]["value"])
    # supernodal tree
    lab = {tuple(v): i + 1 for i, v in enumerate(FIG1["supernodes_maximal"]["value"])}
    got = {}
    for J in range(o.nsuper):
        if s["sparent"][J] >= 0:
            got[str(lab[tuple(sets[J])])] = lab[tuple(sets[s["sparent"][J]])]
    assert got == FIG1["supernodal_tree"]["value"]
    # panel shapes J1 5x2, J3 6x3 (m x k)
    for jl, (m, k) in FIG1["panel_shapes"]["value"].items():
        J = sets.index(FIG1["supernodes_maximal"]["value"][int(jl) - 1])
        assert s["rows_ptr"][J + 1] - s["rows_ptr"][J] == m
        assert s["sfirst"][J + 1] - s["sfirst"][J] == k
    # relind(J3,J6) = [2,1,0] and relind(J1,J6) = [1]
    def relind(Jl, Pl):
        J = sets.index(FIG1["supernodes_maximal"]["value"][Jl - 1])
        P = sets.index(FIG1["supernodes_maximal"]["value"][Pl - 1])
        for q in range(s["rel_ptr"][J], s["rel_ptr"][J + 1]):
            if s["rel_anc"][q] == P:
                return s["relind"][s["rel_off"][q]:s["rel_off"][q + 1]].tolist()
        return None
    assert relind(3, 6) == FIG1["relind"]["J3_J6"]
    assert relind(1, 6) == FIG1["relind"]["J1_J6"]


def test_fig1_update_matrix_support():
    """U_J1 = L_{R,J1} L_{R,J1}^T has exactly the Fig. 2 support."""
    p = fig1_problem()
    o = oracle.Oracle.from_problem(p, cap=-1, rule=1)
    s = o.symbolic()
    assert o.factor() == -1
    L = dense_of(o.L_csc(), 15)
    inv = np.argsort(s["perm_final"])          # final -> paper label - 1
    cols = [int(s["perm_final"][c - 1]) for c in (1, 2)]
    rows = [r for r in range(15) if r not in cols and np.any(L[r, cols] != 0)]
    LR = L[np.ix_(rows, cols)]
    U = LR @ LR.T
    support = sorted((int(inv[rows[a]]) + 1, int(inv[rows[b]]) + 1)
                     for a in range(len(rows)) for b in range(len(rows))
                     if U[a, b] != 0 and inv[rows[a]] >= inv[rows[b]])
    assert support == sorted(map(tuple, FIG1["U_J1_support"]["value"]))


def test_fig1_rlb_blocks():
    """RLB blocks of J1: B = {6,7} inside J3 and B' = {14} inside J6."""
    p = fig1_problem()
    o = oracle.Oracle.from_problem(p, cap=-1, rule=1)
    s = o.symbolic()
    inv = np.argsort(s["perm_final"])
    lab = lambda c: int(inv[c]) + 1
    blocks = {}
    for J in range(o.nsuper):
        cols = tuple(sorted(lab(c) for c in range(s["sfirst"][J], s["sfirst"][J + 1])))
        rows = s["rows"][s["rows_ptr"][J]:s["rows_ptr"][J + 1]]
        blocks[cols] = [[lab(r) for r in rows[s["blk_q"][b]:s["blk_q"][b] + s["blk_len"][b]]]
                        for b in range(s["blk_ptr"][J], s["blk_ptr"][J + 1])]
    assert blocks[(1, 2)] == [[6, 7], [14]]
    assert blocks[(3, 4)] == [[8, 9], [13]]     # SPEC S:229 derived example
    assert blocks[(12, 13, 14, 15)] == []


def test_fig1_merge_costs_spec():
    """SPEC S:181 costs on the Fig. 1 partition: the first greedy pick is (J2,J4) at cost 2."""
    p = fig1_problem()
    o = oracle.Oracle.from_problem(p, cap=10.0, rule=1)
    s = o.symbolic()
    child, parent, cost = s["merges"][0]
    assert cost == FIG1["first_merge_costs_maximal"]["value"]["2-4"] == 2


def test_fig1_fundamental_partition_and_merge_trace():
    p = fig1_problem()
    o = oracle.Oracle.from_problem(p, cap=0.25, rule=0)
    s = o.symbolic()
    post = s["post"]
    lab = lambda new: int(post[new]) + 1
    fund = [[lab(c) for c in range(s["ffirst"][f], s["ffirst"][f + 1])] for f in range(o.nfund)]
    assert sorted(map(sorted, fund)) == sorted(map(sorted, FIG1["fundamental_partition"]["value"]))
    assert o.nnzL == 57
    # trace: (child group columns) -> (parent group columns), cost; groups grow as merges apply
    groups = {f: set(fund[f]) for f in range(o.nfund)}
    trace = []
    for c, pgrp, cost in s["merges"]:
        trace.append([sorted(groups[c]), sorted(groups[pgrp]), cost])
        groups[pgrp] |= groups.pop(c)
    assert trace == [[sorted(a), sorted(b), c] for a, b, c in FIG1["merge_trace_fundamental_cap025"]["value"]]
    assert o.added == 13
    final = []
    for J in range(o.nsuper):
        final.append([int(np.where(s["perm_final"] == c)[0][0]) + 1 for c in range(s["sfirst"][J], s["sfirst"][J + 1])])
    assert final == FIG1["final_order_fundamental_cap025"]["value"]


# ---------------------------------------------------------------- brute force on tiny inputs
def brute_symbolic(C):
    """Dense boolean elimination: struct of L for the SPD pattern of C (no cancellation)."""
    n = C.shape[0]
    M = C != 0
    for j in range(n):
        nz = [i for i in range(j + 1, n) if M[i, j]]
        for a in nz:
            for b in nz:
                if a >= b:
                    M[a, b] = True
    cc = [1 + sum(1 for i in range(j + 1, n) if M[i, j]) for j in range(n)]
    par = [min([i for i in range(j + 1, n) if M[i, j]], default=-1) for j in range(n)]
    return np.tril(M), cc, par


@pytest.mark.parametrize("trial", range(0, 160))
def test_random_corpus_symbolic_and_numeric(trial):
    p = gen.random_spd(trial)
    o = oracle.Oracle.from_problem(p, cap=0.25)
    s = o.symbolic()
    pf = s["perm_final"]
    C = permuted_dense(p, pf)
    M, cc, par = brute_symbolic(C)
    assert s["cc_final"].tolist() == cc
    assert s["parent_final"].tolist() == par
    assert o.nnzL == sum(cc)
    assert o.flops == float(sum(c * c for c in cc))
    # numeric vs LAPACK (numpy) dense Cholesky
    assert o.factor() == -1
    L = dense_of(o.L_csc(), p.n)
    Lref = np.linalg.cholesky(C)
    assert np.abs(L - Lref).max() <= 1e-13 * max(1.0, np.abs(Lref).max())
    # LAPACK's factor is zero outside the symbolic pattern (no numerical cancellation here)
    assert np.all(Lref[~M] == 0.0)
    check_invariants(o, s, p.n, 0.25, Lref)


def check_invariants(o, s, n, cap, Lref=None):
    sf, rp, rows = s["sfirst"], s["rows_ptr"], s["rows"]
    ns = o.nsuper
    snode = np.empty(n, int)
    for J in range(ns):
        snode[sf[J]:sf[J + 1]] = J
    # etree: parent > child; containment: struct(L_j)\{j} subset of struct(L_parent(j))
    par = s["parent_final"]
    assert np.all((par == -1) | (par > np.arange(n)))
    # supernodes: rows begin with own columns, sorted, contiguous columns
    storage = 0
    for J in range(ns):
        k = sf[J + 1] - sf[J]
        r = rows[rp[J]:rp[J + 1]]
        m = len(r)
        assert np.all(np.diff(r) > 0)
        assert r[:k].tolist() == list(range(sf[J], sf[J + 1]))
        storage += k * m - k * (k - 1) // 2
        # sparent = snode of the parent of the last column
        last = sf[J + 1] - 1
        assert s["sparent"][J] == (-1 if par[last] == -1 else snode[par[last]])
        # relind: strictly decreasing, and rows(P)[m_P-1-relind] == rows(J)[q]
        for q in range(s["rel_ptr"][J], s["rel_ptr"][J + 1]):
            P = s["rel_anc"][q]
            q0 = s["rel_q0"][q]
            rel = s["relind"][s["rel_off"][q]:s["rel_off"][q + 1]]
            rP = rows[rp[P]:rp[P + 1]]
            assert len(rel) == m - q0
            assert np.all(np.diff(rel) < 0)
            assert rP[len(rP) - 1 - rel].tolist() == r[q0:].tolist()
            assert r[q0] >= sf[P] and (q0 == k or r[q0 - 1] < sf[P])
    # RLB blocks: disjoint, ordered, cover R_J; each a run of consecutive global rows
    # inside one ancestor's columns, maximal; relindB = relind(J,P) of its first row
    for J in range(ns):
        k = sf[J + 1] - sf[J]
        r = rows[rp[J]:rp[J + 1]]
        q = k
        for b in range(s["blk_ptr"][J], s["blk_ptr"][J + 1]):
            assert s["blk_q"][b] == q
            blk = r[q:q + s["blk_len"][b]]
            assert len(blk) >= 1 and np.all(np.diff(blk) == 1)
            P = s["blk_anc"][b]
            assert np.all((blk >= sf[P]) & (blk < sf[P + 1]))
            rP = rows[rp[P]:rp[P + 1]]
            assert rP[len(rP) - 1 - s["blk_relind"][b]] == blk[0]
            q += len(blk)
            if q < len(r):       # maximal: the next row breaks the run or changes ancestor
                assert r[q] != r[q - 1] + 1 or not (sf[P] <= r[q] < sf[P + 1])
        assert q == len(r)
    # merged storage growth == sum of merge costs, never above the cap
    assert storage - o.nnzL == o.added == sum(c for _, _, c in s["merges"])
    assert o.added <= cap * o.nnzL + 1e-9
    # stopping rule is exact: no remaining child-parent merge fits in the budget
    m_of = lambda J: rp[J + 1] - rp[J]
    k_of = lambda J: sf[J + 1] - sf[J]
    rem = [k_of(J) * (k_of(J) + m_of(s["sparent"][J]) - m_of(J)) for J in range(ns) if s["sparent"][J] >= 0]
    if rem and cap >= 0:
        assert o.added + min(rem) > cap * o.nnzL
    if Lref is not None:
        # every exact nonzero lies in its supernode's panel; padding is exactly zero in LAPACK's L
        inpanel = np.zeros((n, n), bool)
        for J in range(ns):
            r = rows[rp[J]:rp[J + 1]]
            for c in range(sf[J], sf[J + 1]):
                inpanel[r[r >= c], c] = True
        assert np.all(inpanel[np.tril(Lref) != 0])


def test_grid_symbolic_invariants_and_padding_zero():
    """A 2D/3D grid with real amalgamation padding: LAPACK's factor is exactly 0 on the padding."""
    for p in (gen.make("T1"), gen.make("T3"), gen.make("T2"), gen.make("C1")):
        o = oracle.Oracle.from_problem(p)
        s = o.symbolic()
        C = permuted_dense(p, s["perm_final"])
        Lref = np.linalg.cholesky(C)
        check_invariants(o, s, p.n, 0.25, Lref)
        assert o.factor() == -1
        L = dense_of(o.L_csc(), p.n)
        assert np.abs(L - Lref).max() <= 1e-12 * np.abs(Lref).max()
        # padding: panel entries outside the exact pattern are exactly 0 in LAPACK's factor
        Lp, Li, _ = o.L_csc()
        pattern = dense_of((Lp, Li, None), p.n) != 0
        sf, rp, rows = s["sfirst"], s["rows_ptr"], s["rows"]
        npad = 0
        for J in range(o.nsuper):
            r = rows[rp[J]:rp[J + 1]]
            for c in range(sf[J], sf[J + 1]):
                rr = r[r >= c]
                pad = rr[~pattern[rr, c]]
                npad += len(pad)
                assert np.all(Lref[pad, c] == 0.0)
        assert npad == o.added


# ---------------------------------------------------------------- closed forms
def test_1d_laplacian_closed_form():
    """tridiag(-1,2,-1): L_jj = sqrt((j+1)/j), L_{j+1,j} = -sqrt(j/(j+1)) (1-based), det = n+1."""
    n = 200
    D = np.diag(np.full(n, 2.0)) + np.diag(np.full(n - 1, -1.0), -1)
    p = gen.from_dense_lower(D)
    o = oracle.Oracle.from_problem(p)
    s = o.symbolic()
    assert s["perm_final"].tolist() == list(range(n))  # a chain is already a postorder
    assert o.factor() == -1
    L = dense_of(o.L_csc(), n)
    j = np.arange(1, n + 1, dtype=float)
    assert np.allclose(np.diag(L), np.sqrt((j + 1) / j), rtol=0, atol=1e-15)
    assert np.allclose(np.diag(L, -1), -np.sqrt(j[:-1] / (j[:-1] + 1)), rtol=0, atol=1e-15)
    assert abs(2 * np.log(np.diag(L)).sum() - math.log(n + 1)) < 1e-12


def grid_logdet(kind, grid, dof):
    """log det of the Dirichlet grid operator from its eigenvalues (closed form)."""
    cs = [np.cos(np.pi * np.arange(1, K + 1) / (K + 1)) for K in grid]
    if kind == 5:
        lam = 4 - 2 * cs[0][None, :] - 2 * cs[1][:, None]
    elif kind == 9:
        lam = 9 - (1 + 2 * cs[0][None, :]) * (1 + 2 * cs[1][:, None])
    elif kind == 7:
        lam = 6 - 2 * (cs[0][None, None, :] + cs[1][None, :, None] + cs[2][:, None, None])
    elif kind == 27:
        lam = 27 - (1 + 2 * cs[0][None, None, :]) * (1 + 2 * cs[1][None, :, None]) * (1 + 2 * cs[2][:, None, None])
    ld = math.fsum(np.log(lam).ravel().tolist())
    if dof == 3:
        ld = 3 * ld + lam.size * math.log(20.0)   # A = K27 (x) B, det B = 5*2*2
    return ld


def test_logdet_closed_form_printed_C1():
    # SURVEY §8(c) prints C1's closed form 1065.0006883542344
    assert abs(grid_logdet(5, (30, 30), 1) - 1065.0006883542344) < 1e-9


@pytest.mark.parametrize("name", ["C1", "T1", "T2", "T3", "S2", "S4", "S5"])
def test_oracle_logdet_matches_closed_form(name):
    p = gen.make(name)
    o = oracle.Oracle.from_problem(p)
    assert o.factor() == -1
    Lp, Li, Lx = o.L_csc()
    ld = 2.0 * math.fsum(np.log(Lx[Lp[:-1]]).tolist())
    ref = grid_logdet(p.kind, p.grid if p.kind not in (5, 9) else p.grid[:2], p.dof)
    assert abs(ld - ref) <= 1e-10 * abs(ref)


# ---------------------------------------------------------------- SPEC tiny examples, failure, solve
def test_spec_tiny_potrf_and_solve():
    # potrf [[4,.],[2,5]] -> [[2,.],[1,2]]; forward/backward with that L
    p = gen.from_dense_lower(np.array([[4.0, 0.0], [2.0, 5.0]]))
    o = oracle.Oracle.from_problem(p)
    assert o.factor() == -1
    assert dense_of(o.L_csc(), 2).tolist() == [[2.0, 0.0], [1.0, 2.0]]
    x = o.solve(np.array([6.0, 7.0]))      # A x = b with x = [1, 1]
    assert np.allclose(x, [1.0, 1.0], atol=1e-15)
    # [[1,.],[2,1]] is not SPD: second pivot 1 - 4 < 0
    q = gen.from_dense_lower(np.array([[1.0, 0.0], [2.0, 1.0]]))
    assert oracle.Oracle.from_problem(q).factor() == 1


def test_not_spd_first_failing_column():
    """Reading R8: C_f(j0,j0) := -1 fails exactly at j0 (pivot <= -1 - sum of squares < 0)."""
    p = gen.make("T3")
    o = oracle.Oracle.from_problem(p)
    s = o.symbolic()
    for j0 in (0, 17, p.n // 2, p.n - 1):
        i0 = int(np.where(s["perm_final"] == j0)[0][0])        # original index of final column j0
        vals = p.values.copy()
        vals[p.colptr[i0]] = -1.0                               # diagonal entry is first in its column
        q = gen.Problem(p.name, p.n, p.colptr, p.rowidx, vals, p.perm)
        assert oracle.Oracle.from_problem(q).factor() == j0


@pytest.mark.parametrize("name", ["C1", "T2", "S2", "S4"])
def test_oracle_solve_backward_error(name):
    p = gen.make(name)
    xstar, b = gen.rhs(p)
    o = oracle.Oracle.from_problem(p)
    assert o.factor() == -1
    x = o.solve(b)
    r = gen.symv(p, x=x) - b
    Anorm = np.abs(gen.to_dense(p)).sum(axis=1).max() if p.n <= 2000 else None
    if Anorm is None:
        rowsum = np.zeros(p.n)
        np.add.at(rowsum, p.rowidx, np.abs(p.values))
        cols = np.repeat(np.arange(p.n), np.diff(p.colptr))
        off = p.rowidx != cols
        np.add.at(rowsum, cols[off], np.abs(p.values[off]))
        Anorm = rowsum.max()
    assert np.abs(r).max() / (Anorm * np.abs(x).max()) <= 1e-12


@pytest.mark.parametrize("name", ["C1", "S2", "S4", "S5", "T2"])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_parallel_oracle_bit_identical(name, threads):
    """The level-parallel O9 build (the timed CPU baseline) computes every column with the
    serial build's operations in the same order: L is bitwise equal, on any thread count."""
    p = gen.make(name)
    a = oracle.Oracle.from_problem(p)
    assert a.factor() == -1
    La = a.L_csc()[2].copy()
    b = oracle.Oracle.from_problem(p)
    assert b.factor(threads=threads) == -1
    assert np.array_equal(La, b.L_csc()[2])


@pytest.mark.parametrize("threads", [1, 4])
def test_parallel_oracle_not_spd(threads):
    """The parallel build reports the serial build's first failing column (recipe R8)."""
    p = gen.make("S4")
    a = oracle.Oracle.from_problem(p)
    pf = a.symbolic()["perm_final"]
    for frac in (0.1, 0.6, 0.99):
        j0 = int(frac * (p.n - 1))
        i0 = int(np.where(pf == j0)[0][0])
        vals = p.values.copy()
        vals[p.colptr[i0]] = -1.0
        q = gen.Problem(p.name, p.n, p.colptr, p.rowidx, vals, p.perm)
        assert oracle.Oracle.from_problem(q).factor() == j0
        assert oracle.Oracle.from_problem(q).factor(threads=threads) == j0


# ---------------------------------------------------------------- O7b partition refinement (R14)
def test_fig1_partition_refinement():
    """Hand-derived refined column order of Fig. 1's cap-0.25 supernodes (tests/golden/fig1.json)."""
    p = fig1_problem()
    o = oracle.Oracle.from_problem(p, cap=0.25, rule=0, pr=1)
    s = o.symbolic()
    final = []
    for J in range(o.nsuper):
        final.append([int(np.where(s["perm_final"] == c)[0][0]) + 1 for c in range(s["sfirst"][J], s["sfirst"][J + 1])])
    assert final == FIG1["partition_refinement_cap025"]["value"]


@pytest.mark.parametrize("trial", range(0, 60))
def test_partition_refinement_random_corpus(trial):
    """PR only reorders columns inside the supernodes (same partition, same column sets); the exact
    structure of the refined order matches dense boolean elimination; the factor matches LAPACK; the
    exact pattern stays inside the panels; relind / RLB invariants hold; and the first refining set of
    every supernode ends up as a prefix of its columns."""
    p = gen.random_spd(2000 + trial)
    o0 = oracle.Oracle.from_problem(p, cap=0.25)
    o = oracle.Oracle.from_problem(p, cap=0.25, pr=1)
    s0, s = o0.symbolic(), o.symbolic()
    assert np.array_equal(s0["sfirst"], s["sfirst"]) and np.array_equal(s0["sparent"], s["sparent"])
    ip0, ip = np.argsort(s0["perm_final"]), np.argsort(s["perm_final"])
    sf = s["sfirst"]
    for J in range(o.nsuper):
        assert sorted(ip0[sf[J]:sf[J + 1]]) == sorted(ip[sf[J]:sf[J + 1]])
    C = permuted_dense(p, s["perm_final"])
    M, cc, par = brute_symbolic(C)
    assert s["cc_final"].tolist() == cc and s["parent_final"].tolist() == par
    assert o.nnzL == sum(cc)
    assert o.factor() == -1
    L = dense_of(o.L_csc(), p.n)
    Lref = np.linalg.cholesky(C)
    assert np.abs(L - Lref).max() <= 1e-13 * max(1.0, np.abs(Lref).max())
    assert np.all(Lref[~M] == 0.0)
    rp, rows = s["rows_ptr"], s["rows"]
    inpanel = np.zeros((p.n, p.n), bool)
    for J in range(o.nsuper):
        r = rows[rp[J]:rp[J + 1]]
        for c in range(sf[J], sf[J + 1]):
            inpanel[r[r >= c], c] = True
    assert np.all(inpanel[np.tril(Lref) != 0])
    # first refining set of each supernode P = its columns in R_J of the smallest such J: a prefix
    snode = np.repeat(np.arange(o.nsuper), np.diff(sf))
    seen = set()
    for J in range(o.nsuper):
        R = rows[rp[J] + (sf[J + 1] - sf[J]):rp[J + 1]]
        for P in np.unique(snode[R]):
            if P in seen:
                continue
            seen.add(P)
            SJ = np.sort(R[snode[R] == P])
            assert SJ.tolist() == list(range(sf[P], sf[P] + len(SJ)))
    # relind and RLB block invariants in the refined numbering
    for J in range(o.nsuper):
        r = rows[rp[J]:rp[J + 1]]
        for q in range(s["rel_ptr"][J], s["rel_ptr"][J + 1]):
            P, q0 = s["rel_anc"][q], s["rel_q0"][q]
            rel = s["relind"][s["rel_off"][q]:s["rel_off"][q + 1]]
            rP = rows[rp[P]:rp[P + 1]]
            assert np.all(np.diff(rel) < 0) and rP[len(rP) - 1 - rel].tolist() == r[q0:].tolist()
        for b in range(s["blk_ptr"][J], s["blk_ptr"][J + 1]):
            blk = r[s["blk_q"][b]:s["blk_q"][b] + s["blk_len"][b]]
            assert np.all(np.diff(blk) == 1)
