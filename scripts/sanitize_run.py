"""One factor + solve of a small config through the C ABI, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck): python scripts/sanitize_run.py NAME [small_max_k]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402

name = sys.argv[1]
small = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p = gen.make(name)
with sp.Solver.from_problem(p, small_max_k=small, use_graph=0) as h:
    assert h.spchol_factor() == (-1, -1)
    xs, b = gen.rhs(p)
    x = h.spchol_solve(b)
    print(name, "small_max_k", small, "backward error", gen.backward_error(p, x, b))
