"""Memory-capped mode (f-4) at full size: factor and solve time with the factor's device storage capped
(GB), against the resident run; closed-form log det and backward error as checks.
python scripts/capped_bench.py C5 16 [C4 8 ...]  -> one JSON line per run."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402
from test_oracle_pins import grid_logdet  # noqa: E402

args = sys.argv[1:] or ["C5", "16"]
for name, gb in zip(args[::2], args[1::2]):
    p = gen.make(name)
    for cap in (0, int(float(gb) * 1e9)):
        with sp.Solver.from_problem(p, device_mem_cap=cap) as h:
            s = torch.cuda.Stream()
            h.spchol_set_stream(s.cuda_stream)
            for _ in range(2):
                h.spchol_factor()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(3):
                h.spchol_factor_async()
            e1.record(s)
            h.spchol_factor_status()
            fms = e0.elapsed_time(e1) / 3
            xs, b = gen.rhs(p)
            d_b = torch.from_numpy(b).cuda()
            d_x = torch.empty_like(d_b)
            h.spchol_solve_device(d_b.data_ptr(), d_x.data_ptr())
            torch.cuda.synchronize()
            e0.record(s)
            h.spchol_solve_device(d_b.data_ptr(), d_x.data_ptr())
            e1.record(s)
            torch.cuda.synchronize()
            sms = e0.elapsed_time(e1)
            x = d_x.cpu().numpy()
            ld = 2.0 * math.fsum(np.log(h.spchol_export_diagonal()).tolist())
            grid = p.grid if p.kind not in (5, 9) else p.grid[:2]
            ref = grid_logdet(p.kind, grid, p.dof)
            rec = {"config": name, "cap_GB": cap / 1e9, "arena_GB": h.query("ARENA_BYTES") / 1e9,
                   "device_GB": h.query("DEVICE_BYTES") / 1e9, "batches": h.query("NBATCHES"),
                   "host_GB": h.query("HOST_BYTES") / 1e9, "factor_ms": fms, "solve_ms": sms,
                   "gflops": h.query("FLOPS_EXACT") / fms / 1e6, "logdet_rel_err": abs(ld - ref) / abs(ref),
                   "backward_error": gen.backward_error(p, x, b)}
            print(json.dumps(rec), flush=True)
