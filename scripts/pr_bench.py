"""Partition refinement (f-2): RLB block count and factor time, RL and RLB, with and without PR.
python scripts/pr_bench.py C3 C4 ...  -> one JSON line per (config, update_mode, pr)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402

for name in sys.argv[1:] or ["C3", "C4"]:
    p = gen.make(name)
    for mode in (0, 1):
        for pr in (0, 1):
            with sp.Solver.from_problem(p, update_mode=mode, partition_refinement=pr) as h:
                s = torch.cuda.Stream()
                h.spchol_set_stream(s.cuda_stream)
                for _ in range(3):
                    h.spchol_factor()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(s)
                for _ in range(3):
                    h.spchol_factor_async()
                e1.record(s)
                h.spchol_factor_status()
                ms = e0.elapsed_time(e1) / 3
                xs, b = gen.rhs(p)
                x = h.spchol_solve(b)
                print(json.dumps({"config": name, "update_mode": ["RL", "RLB"][mode], "pr": pr,
                                  "rlb_blocks": h.query("NBLOCKS"), "nnz_L_exact": h.query("NNZ_L"),
                                  "flops_exact": h.query("FLOPS_EXACT"), "factor_ms": ms,
                                  "backward_error": gen.backward_error(p, x, b)}), flush=True)
