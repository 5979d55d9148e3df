"""Serialized per-(level, kernel class) time of one factor (kernel timing mode, CUDA events per launch).
python scripts/level_kernels.py C4"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402

names = {v: k for k, v in sp.KERNEL_KINDS.items()}
for name in sys.argv[1:] or ["C4"]:
    p = gen.make(name)
    with sp.Solver.from_problem(p) as h:
        h.spchol_factor()
        h.spchol_enable_kernel_timing(True)
        h.spchol_factor()
        tr = h.spchol_kernel_trace()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, l, n, ms in zip(tr["kinds"], tr["levels"], tr["ntasks"], tr["ms"]):
        a = agg[(int(l), names[int(k)])]
        a[0] += 1
        a[1] += ms
    print(name)
    for l in sorted({k[0] for k in agg}):
        row = {kk: "%d/%.2f" % tuple(v) for (ll, kk), v in agg.items() if ll == l}
        print("  level", l, row)
