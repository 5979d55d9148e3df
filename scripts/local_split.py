import os, sys, json, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, gen, paper_2409_14009_b200 as sp
p = gen.make(sys.argv[1] if len(sys.argv) > 1 else "C4")
h = sp.Solver.from_problem(p)
h.spchol_factor(); h.spchol_factor()
h.spchol_enable_kernel_timing(True)
h.spchol_factor_async()
tr = h.spchol_kernel_trace()
st = h.spchol_kernel_stats("local_update")
# plan flops per launch are not exported; estimate K from ms/tasks is not possible -> use ntasks and ms
ks = collections.defaultdict(lambda: [0, 0.0, 0])
for k, l, n, t in zip(tr["kinds"], tr["levels"], tr["ntasks"], tr["ms"]):
    if k == 3:
        b = "n<=148" if n <= 148 else ("n<=592" if n <= 592 else ("n<=4096" if n <= 4096 else "n>4096"))
        ks[b][0] += 1; ks[b][1] += t; ks[b][2] += n
for b, v in sorted(ks.items()):
    print(b, "launches", v[0], "ms %.2f" % v[1], "tasks", v[2], "us/task %.2f" % (1e3 * v[1] / v[2]))
print("local total", st)
