"""Per-launch kernel trace (serialized timing) of the launches of given levels of one config."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import paper_2409_14009_b200 as sp

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--levels", default="0")
a = ap.parse_args()
h = sp.Solver.from_problem(gen.make(a.config))
h.spchol_factor()
h.spchol_enable_kernel_timing(True)
h.spchol_factor_async()
tr = h.spchol_kernel_trace()
names = {v: k for k, v in sp.KERNEL_KINDS.items()}
want = {int(x) for x in a.levels.split(",")}
for k, l, n, t in zip(tr["kinds"], tr["levels"], tr["ntasks"], tr["ms"]):
    if int(l) in want:
        print(int(l), names[int(k)], int(n), round(float(t) * 1e3, 1))
