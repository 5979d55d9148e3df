"""One factor, then one solve of a config (the command the solve launch-list capture wraps):
python scripts/one_solve.py C4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
p = gen.make(name)
with sp.Solver.from_problem(p, use_graph=0) as h:
    h.spchol_factor()
    xs, b = gen.rhs(p)
    x = h.spchol_solve(b)
    print(name, "backward error", gen.backward_error(p, x, b))
