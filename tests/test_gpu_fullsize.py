"""Full-size BASELINE configs on the GPU (-m gpu): properties that hold at any size, in the launch
configuration bench.py times (CUDA graph): log det of the grid operator from its closed-form
eigenvalues (pins the whole diagonal of L), normwise backward error of the solve,
and the symbolic arrays against the oracle's golden digests."""
import hashlib
import json
import os

import numpy as np
import pytest

import gen
import paper_2409_14009_b200 as sp
from helpers import logdet_from_diag
from test_oracle_pins import grid_logdet

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_fullsize_config(name):
    p = gen.make(name)
    with sp.Solver.from_problem(p) as h:
        gpath = os.path.join(HERE, "golden", f"symbolic_{name}.json")
        if os.path.exists(gpath):
            g = json.load(open(gpath))
            sym = h.spchol_export_symbolic()
            for k in ("perm_final", "sfirst", "rows", "relind"):
                assert hashlib.sha256(np.ascontiguousarray(sym[k]).tobytes()).hexdigest() == g["sha256"][k], k
        h.spchol_factor()
        h.spchol_factor()                       # graph replay
        diag = h.spchol_export_diagonal()
        ld = logdet_from_diag(diag)
        grid = p.grid if p.kind not in (5, 9) else p.grid[:2]
        ref = grid_logdet(p.kind, grid, p.dof)
        assert abs(ld - ref) <= 1e-10 * abs(ref), (ld, ref)
        xs, b = gen.rhs(p)
        x = h.spchol_solve(b)
        berr = gen.backward_error(p, x, b)
        assert berr <= 1e-12, berr
        print(name, "logdet rel err %.2e  backward error %.2e  forward err %.2e" %
              (abs(ld - ref) / abs(ref), berr, np.abs(x - xs).max() / np.abs(xs).max()))


@pytest.mark.parametrize("name,N", [("C2", 3000), ("C3", 3000), ("C4", 4000), ("C5", 3000)])
def test_fullsize_leading_block_factor(name, N):
    """Sampled full-size parity in the bench configuration (CUDA graph, replayed): the first N
    columns of the nested-dissection order are whole subtrees, so the factor restricted to them
    (in the final order) is exactly the Cholesky factor of that principal block of P_f A P_f^T,
    computed independently here by a dense LAPACK Cholesky; every entry is compared (tolerance
    of the north_star, max|dL| / max|L| <= 1e-10)."""
    p = gen.make(name)
    with sp.Solver.from_problem(p) as h:
        h.spchol_factor()
        h.spchol_factor()
        sym = h.spchol_export_symbolic()
        pf, sfirst, rows_ptr, rows = sym["perm_final"], sym["sfirst"], sym["rows_ptr"], sym["rows"]
        off, ld, _ = h.spchol_export_panels(values=False)
        idx = np.where(p.perm < N)[0]                    # leading ND block: closed under descendants
        order = idx[np.argsort(pf[idx])]                 # its columns in final order
        f = pf[order]
        pos = -np.ones(p.n, np.int64)
        pos[f] = np.arange(N)
        Lg = np.zeros((N, N))
        for J in np.unique(np.searchsorted(sfirst, f, side="right") - 1):
            k, m = int(sfirst[J + 1] - sfirst[J]), int(rows_ptr[J + 1] - rows_ptr[J])
            buf = np.empty(int(ld[J]) * k, np.float64)
            assert h._L.spchol_export_panel(h._h, int(J), sp._vp(buf)) == 0
            P = buf.reshape(k, int(ld[J])).T[:m]
            rJ = rows[rows_ptr[J]:rows_ptr[J + 1]]
            for c in range(k):
                col = int(sfirst[J]) + c
                if pos[col] < 0:
                    continue
                sel = (pos[rJ] >= 0) & (rJ >= col)
                Lg[pos[rJ[sel]], pos[col]] = P[sel, c]
    # the principal block of A in the same order, from A's stored lower triangle (caller numbering)
    po = -np.ones(p.n, np.int64)
    po[order] = np.arange(N)
    A = np.zeros((N, N))
    for j in order:
        r = p.rowidx[p.colptr[j]:p.colptr[j + 1]]
        v = p.values[p.colptr[j]:p.colptr[j + 1]]
        keep = po[r] >= 0
        A[po[r[keep]], po[j]] = v[keep]
        A[po[j], po[r[keep]]] = v[keep]
    Lref = np.linalg.cholesky(A)
    err = np.abs(Lg - Lref).max() / np.abs(Lref).max()
    assert err <= 1e-10, err


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize_top_levels_llt(name):
    """Exact-result check at full size where most of the flops live: for sampled
    columns j of every supernode in the top three levels (the root chain and the largest separators),
    every stored entry (L L^T)(i, j), i >= j, computed from the exported panels, equals C_f(i, j)
    = (P_f A P_f^T)(i, j) to 1e-12 max|A| — independent of the oracle and of the kernels, in the bench
    configuration (CUDA graph, replayed)."""
    from helpers import llt_sample_error, top_level_columns
    p = gen.make(name)
    with sp.Solver.from_problem(p) as h:
        h.spchol_factor()
        h.spchol_factor()
        sym = h.spchol_export_symbolic()
        off, ld, pan = h.spchol_export_panels()
    cols = top_level_columns(sym, nlev=3, per_sn=3)
    err, cnt = llt_sample_error(p, sym, off, ld, pan, cols)
    print(name, "sampled columns", len(cols), "entries", cnt, "max |LL^T - C_f| / max|A|", err)
    assert cnt >= 10 ** 5 if name != "C3" else cnt >= 10 ** 4
    assert err <= 1e-12, err
