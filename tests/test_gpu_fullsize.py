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
