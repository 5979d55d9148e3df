"""One multi-rank factor + solve through the library's real NCCL code path, every rank a thread of
this process on one GPU, NCCL replaced by tests/mock_nccl (SPCHOL_NCCL_LIB).  Run as a subprocess
by tests/test_gpu_parity.py::test_distributed_nccl_path_mock; prints one JSON line."""
import json
import os
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
os.environ["SPCHOL_NCCL_LIB"] = os.path.join(HERE, "mock_nccl", "libmocknccl.so")

import numpy as np  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402
from helpers import (backward_error, llt_sample_error, logdet_from_diag, lower_panel_mask,  # noqa: E402
                     panel_index_of_pattern, top_level_columns)


def main_not_spd(name, world, frac):
    """Rank-local pivot failure: every rank must report the same first failing column (the
    all-reduce(min) of the fail flags), in the final and the caller's numbering."""
    p = gen.make(name)
    with sp.Solver.from_problem(p, device=-1) as h0:
        pf = h0.spchol_export_symbolic()["perm_final"]
    j0 = int(frac * (p.n - 1))
    i0 = int(np.where(pf == j0)[0][0])
    vals = p.values.copy()
    vals[p.colptr[i0]] = -1.0
    q = gen.Problem(p.name, p.n, p.colptr, p.rowidx, vals, p.perm)
    expect = oracle.Oracle.from_problem(q).factor()
    uid = sp.spchol_dist_nccl_unique_id()
    hs = [sp.Solver.from_problem(q, dist_world=world, dist_rank=r) for r in range(world)]
    got = [None] * world

    def run(r):
        try:
            hs[r].spchol_dist_attach_nccl(uid)
            hs[r].spchol_factor()
            got[r] = "no error"
        except sp.NotSPDError as e:
            got[r] = (e.fail_col, e.fail_col_orig)
        except Exception as e:  # noqa: BLE001
            got[r] = repr(e)

    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if any(t.is_alive() for t in th):
        print(json.dumps({"ok": False, "why": "hang"}), flush=True)
        os._exit(3)
    ok = expect == j0 and all(g == (j0, i0) for g in got)
    print(json.dumps({"ok": ok, "expect": [j0, i0], "oracle": expect, "got": [list(g) if isinstance(g, tuple) else g
                                                                            for g in got]}), flush=True)


def main(name, world, nrounds=2, check_panels=True, full=False):
    """Factor + solve `nrounds` times on `world` rank threads; every rank holds only its own part of L
    (the sum of the ranks' panel exports is L), checked against the oracle."""
    prob = gen.make(name)
    pr = int(os.environ.get("MOCK_PR", "0"))
    uid = sp.spchol_dist_nccl_unique_id()
    hs = [sp.Solver.from_problem(prob, dist_world=world, dist_rank=r, partition_refinement=pr) for r in range(world)]
    xs, b = gen.rhs(prob)
    out = [None] * world
    err = [None] * world
    t_factor = [0.0] * world
    multi = [None] * world
    B3 = np.asfortranarray(np.stack([b, np.roll(b, 7), -0.5 * b], axis=1))

    def run(r):
        try:
            h = hs[r]
            h.spchol_dist_attach_nccl(uid)
            res = []
            for _ in range(nrounds):                 # factor again: the second reuses every plan
                t0 = time.time()
                h.spchol_factor()
                t_factor[r] = time.time() - t0
                res.append(h.spchol_solve(b))
            multi[r] = h.spchol_solve(B3)            # three right-hand sides in one block
            out[r] = res
        except Exception as e:  # noqa: BLE001
            err[r] = repr(e)

    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=1800)
    if any(t.is_alive() for t in th):
        print(json.dumps({"ok": False, "why": "hang (NCCL call order differs between ranks?)"}), flush=True)
        os._exit(3)
    if any(err):
        print(json.dumps({"ok": False, "why": err}), flush=True)
        return
    berr = max(backward_error(prob, x, b) for res in out for x in res)
    berr = max([berr] + [backward_error(prob, multi[r][:, c], B3[:, c]) for r in range(world) for c in range(3)])
    # every rank receives the whole solution (all-reduce of the masked components): bitwise equal
    ref = out[0][-1]
    same = all(np.array_equal(o[-1], ref) for o in out)
    diag = sum(h.spchol_export_diagonal() for h in hs)
    rec = {"ok": True, "berr": berr, "ranks_agree": bool(same), "ntop_dist": hs[0].query("NTOP_DIST"),
           "markers": hs[0].query("NMARKERS"), "logdet": logdet_from_diag(diag),
           "device_bytes": [h.query("DEVICE_BYTES") for h in hs], "arena_bytes": [h.query("ARENA_BYTES") for h in hs],
           "send_bytes": [h.query("COMM_SEND_BYTES") for h in hs], "recv_bytes": [h.query("COMM_RECV_BYTES") for h in hs],
           "factor_s": max(t_factor)}
    if full:
        # full-size configs: closed-form log det, sampled exact check L L^T = C_f on the top levels
        # (the distributed supernodes), panels summed over the ranks' exports
        from test_oracle_pins import grid_logdet
        grid = prob.grid if prob.kind not in (5, 9) else prob.grid[:2]
        ref = grid_logdet(prob.kind, grid, prob.dof)
        rec["logdet_rel_err"] = abs(rec["logdet"] - ref) / abs(ref)
        s_gpu = hs[0].spchol_export_symbolic()
        off, ld, pan = hs[0].spchol_export_panels()
        for h in hs[1:]:
            pan += h.spchol_export_panels()[2]
        cols = top_level_columns(s_gpu, nlev=3, per_sn=3)
        rec["llt_err"], rec["llt_entries"] = llt_sample_error(prob, s_gpu, off, ld, pan, cols)
        del pan
    elif check_panels:
        o = oracle.Oracle.from_problem(prob, pr=pr)
        assert o.factor() == -1
        Lp, Li, Lx = o.L_csc()
        s_gpu = hs[0].spchol_export_symbolic()
        off, ld, pan = hs[0].spchol_export_panels()
        for h in hs[1:]:
            pan = pan + h.spchol_export_panels()[2]
        idx = panel_index_of_pattern(s_gpu, off, ld, Lp, Li)
        rec["lerr"] = float(np.abs(pan[idx] - Lx).max() / np.abs(Lx).max())
        # padding: every panel entry outside the exact pattern is exactly zero on every rank
        mask = lower_panel_mask(s_gpu, off, ld, len(pan))
        mask[idx] = False
        rec["padding_nonzeros"] = int(np.count_nonzero(pan[mask]))
    print(json.dumps(rec), flush=True)
    for h in hs:
        h.close()


if __name__ == "__main__":
    if len(sys.argv) > 3:
        main_not_spd(sys.argv[1], int(sys.argv[2]), float(sys.argv[3]))
    else:
        full = os.environ.get("MOCK_FULL", "0") == "1"
        main(sys.argv[1], int(sys.argv[2]), nrounds=1 if full else 2, full=full)
