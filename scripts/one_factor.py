"""One factor of a config (analyze, upload, graph capture + one replay-equivalent launch): the command the
ncu captures of round 2 wrap.  python scripts/one_factor.py C4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
p = gen.make(name)
with sp.Solver.from_problem(p) as h:
    h.spchol_factor()
    print(name, "launches per factor", h.query("LAUNCHES"))
