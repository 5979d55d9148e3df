"""Solve throughput with multiple right-hand sides (f-1): device-resident B (n x nrhs), CUDA events,
per call and per right-hand side; GB/s on the exact factor read twice per pass (forward + backward).
python scripts/solve_bench.py C4 [C5 ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402

for name in sys.argv[1:] or ["C4"]:
    p = gen.make(name)
    with sp.Solver.from_problem(p) as h:
        h.spchol_factor()
        s = torch.cuda.Stream()
        h.spchol_set_stream(s.cuda_stream)
        nnzL = h.query("NNZ_L")
        for nrhs in (1, 2, 4, 16):
            B = torch.randn(nrhs, p.n, dtype=torch.float64, device="cuda")
            X = torch.empty_like(B)
            for _ in range(2):
                h.spchol_solve_device(B.data_ptr(), X.data_ptr(), nrhs, p.n)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(5):
                h.spchol_solve_device(B.data_ptr(), X.data_ptr(), nrhs, p.n)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            nb = nrhs // 4 + (nrhs % 4) // 2 + (nrhs % 2)   # blocks of 4 / 2 / 1
            print(json.dumps({"config": name, "nrhs": nrhs, "ms": ms, "ms_per_rhs": ms / nrhs, "passes_over_L": nb,
                              "GBps_L_read_twice_per_pass": nb * 2 * 8 * nnzL / (ms / 1e3) / 1e9}), flush=True)
