"""Diagnostics: where does a multi-rank factor (ranks as threads over tests/mock_nccl) differ from the
single-GPU factor?  Per supernode max |L_dist - L_1gpu| / max |L|, in supernode order."""
import os
import sys
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
os.environ["SPCHOL_NCCL_LIB"] = os.path.join(ROOT, "tests", "mock_nccl", "libmocknccl.so")
import numpy as np  # noqa: E402

import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402

name, world = sys.argv[1], int(sys.argv[2])
if name.startswith("G"):        # G<kind>_<k>: a 3D grid of the given stencil, ND ordered
    kind, k = name[1:].split("_")
    p = gen.make_grid(int(kind), int(k), int(k), int(k))
else:
    p = gen.make(name)
with sp.Solver.from_problem(p) as h1:
    h1.spchol_factor()
    sym = h1.spchol_export_symbolic()
    ns = len(sym["sfirst"]) - 1
    ref = [h1.spchol_export_panel(J) for J in range(ns)]
uid = sp.spchol_dist_nccl_unique_id()
hs = [sp.Solver.from_problem(p, dist_world=world, dist_rank=r) for r in range(world)]
err = [None] * world


def run(r):
    try:
        hs[r].spchol_dist_attach_nccl(uid)
        hs[r].spchol_factor()
    except Exception as e:  # noqa: BLE001
        err[r] = repr(e)


th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
[t.start() for t in th]
[t.join() for t in th]
print("errors:", err)
owner, towner, _, _ = hs[0].spchol_export_mapping(with_top_owner=True)
lvl = sym["level"]
scale = max(np.abs(x).max() for x in ref if x.size)
bad = 0
for J in range(ns):
    got = sum(h.spchol_export_panel(J) for h in hs)
    m = ref[J].shape[0]
    d = np.abs(got[:m] - ref[J][:m]).max() / scale if ref[J].size else 0.0
    if d > 1e-10:
        bad += 1
        if bad <= 25:
            k = ref[J].shape[1]
            cols = np.where(np.abs(got[:m] - ref[J][:m]).max(axis=0) > 1e-10 * scale)[0]
            print(f"J={J} level={lvl[J]} owner={owner[J]} towner={towner[J]} m={m} k={k} err={d:.2e} "
                  f"bad cols {cols[:5]}..{cols[-3:]} ({len(cols)})")
            if owner[J] < 0:
                D = np.abs(got[:m] - ref[J][:m])
                for C in range(0, min(k, 256 * 24), 256):
                    blk = D[:, C:C + 256]
                    rws = np.where(blk.max(axis=1) > 1e-10 * scale)[0]
                    print(f"   block {C // 256}: max {blk.max() / scale:.2e} bad rows {rws[:3]}..{rws[-3:]} ({len(rws)})"
                          f" per-rank nonzero: {[int(np.count_nonzero(h.spchol_export_panel(J)[:m, C:C + 256])) for h in hs]}")
print("bad supernodes", bad, "of", ns, "ntop_dist", hs[0].query("NTOP_DIST"))
