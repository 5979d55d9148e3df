"""Wall time of the factor truncated after each level (SPCHOL_MAX_LEVEL=l, CUDA graph, events): the
difference between consecutive levels is that level's cost in the real overlapped schedule.
python scripts/level_profile.py C2 [C3 ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402


def timed(p, level):
    os.environ["SPCHOL_MAX_LEVEL"] = str(level)
    with sp.Solver.from_problem(p) as h:
        s = torch.cuda.Stream()
        h.spchol_set_stream(s.cuda_stream)
        for _ in range(2):
            h.spchol_factor_async()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            h.spchol_factor_async()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 5, h.query("NLEVELS")


for name in sys.argv[1:] or ["C2"]:
    p = gen.make(name)
    t_prev, out = 0.0, []
    _, nl = timed(p, 0)
    with sp.Solver.from_problem(p, device=-1) as h:
        sym = h.spchol_export_symbolic()
    lvl, sf, rp = sym["level"], sym["sfirst"], sym["rows_ptr"]
    import numpy as np
    k = np.diff(sf).astype(float)
    m = np.diff(rp).astype(float)
    for l in range(nl):
        t, _ = timed(p, l)
        sel = lvl == l
        fl = float(sum(((m[J] - np.arange(int(k[J]))) ** 2).sum() for J in np.where(sel)[0]))
        out.append({"level": l, "ms": t - t_prev, "cum_ms": t, "supernodes": int(sel.sum()), "max_k": int(k[sel].max()),
                    "flops_exec": fl, "TFLOPs": fl / max(t - t_prev, 1e-6) / 1e9})
        t_prev = t
    print(json.dumps({"config": name, "levels": out}), flush=True)
