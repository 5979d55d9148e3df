"""One multi-rank factor + solve through the library's real NCCL code path, every rank a thread of
this process on one GPU, NCCL replaced by tests/mock_nccl (SPCHOL_NCCL_LIB).  Run as a subprocess
by tests/test_gpu_parity.py::test_distributed_nccl_path_mock; prints one JSON line."""
import json
import os
import sys
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
os.environ["SPCHOL_NCCL_LIB"] = os.path.join(HERE, "mock_nccl", "libmocknccl.so")

import numpy as np  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402
from helpers import backward_error, panel_index_of_pattern  # noqa: E402


def main(name, world):
    prob = gen.make(name)
    uid = sp.spchol_dist_nccl_unique_id()
    hs = [sp.Solver.from_problem(prob, dist_world=world, dist_rank=r) for r in range(world)]
    xs, b = gen.rhs(prob)
    out = [None] * world
    err = [None] * world

    def run(r):
        try:
            h = hs[r]
            h.spchol_dist_attach_nccl(uid)
            res = []
            for _ in range(2):                     # factor twice: the second reuses every plan
                h.spchol_factor()
                res.append(h.spchol_solve(b))
            out[r] = res
        except Exception as e:  # noqa: BLE001
            err[r] = repr(e)

    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if any(t.is_alive() for t in th):
        print(json.dumps({"ok": False, "why": "hang (NCCL call order differs between ranks?)"}), flush=True)
        os._exit(3)
    if any(err):
        print(json.dumps({"ok": False, "why": err}), flush=True)
        return
    berr = max(backward_error(prob, x, b) for res in out for x in res)
    # the level solve accumulates with FP64 RED, so ranks agree to rounding, not bitwise
    ref = out[0][0]
    same = all(np.abs(o[k] - ref).max() <= 1e-12 * np.abs(ref).max() for o in out for k in range(2))
    o = oracle.Oracle.from_problem(prob)
    assert o.factor() == -1
    Lp, Li, Lx = o.L_csc()
    s_gpu = hs[0].spchol_export_symbolic()
    off, ld, pan = hs[0].spchol_export_panels()
    idx = panel_index_of_pattern(s_gpu, off, ld, Lp, Li)
    lerr = float(np.abs(pan[idx] - Lx).max() / np.abs(Lx).max())
    print(json.dumps({"ok": True, "berr": berr, "lerr": lerr, "ranks_agree": bool(same),
                      "ntop_dist": hs[0].query("NTOP_DIST"), "markers": hs[0].query("NMARKERS")}), flush=True)
    for h in hs:
        h.close()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
