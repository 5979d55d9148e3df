"""One factorization of a config, for ncu (launch list / --set full captures)."""
import argparse
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import paper_2409_14009_b200 as sp

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--block", type=int, default=0)
a = ap.parse_args()
p = gen.make(a.config)
h = sp.Solver.from_problem(p, use_graph=0, block=a.block)
for _ in range(a.reps):
    h.spchol_factor()
print("ok", a.config, h.query("LAUNCHES"))
