"""The cdiv chain in isolation: a dense SPD matrix is one supernode, so its factor is a pure chain of
64-column steps (POTRF -> TRSM -> in-block update, NEXT / REST lookahead).  Prints the factor time
(CUDA graph, events) against the DMMA bound, and per-launch times of each kernel class (serialized
timing pass).  python scripts/chain_bench.py [n ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402


def dense_problem(n, seed=1):
    rng = np.random.default_rng(seed)
    nnz = n * (n + 1) // 2
    colptr = np.zeros(n + 1, np.int64)
    colptr[1:] = np.cumsum(n - np.arange(n))
    rows = np.concatenate([np.arange(j, n, dtype=np.int32) for j in range(n)])
    vals = -rng.uniform(0.0, 1.0, nnz) / n
    diag_pos = colptr[:-1]
    vals[diag_pos] = 2.0
    return gen.Problem(f"dense{n}", n, colptr, rows, vals, np.arange(n, dtype=np.int32))


for n in [int(x) for x in sys.argv[1:]] or [2048, 4096, 8192]:
    p = dense_problem(n)
    with sp.Solver.from_problem(p) as h:
        for _ in range(3):
            h.spchol_factor()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 10
        s = torch.cuda.Stream()
        h.spchol_set_stream(s.cuda_stream)
        e0.record(s)
        for _ in range(K):
            h.spchol_factor_async()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        fl = h.query("FLOPS_EXEC")
        h.spchol_enable_kernel_timing(True)
        h.spchol_factor()
        st = {k: h.spchol_kernel_stats(k) for k in sp.KERNEL_KINDS}
        h.spchol_enable_kernel_timing(False)
        per = {k: round(1e3 * v["ms"] / v["launches"], 2) for k, v in st.items() if v["launches"]}
        print(json.dumps({"n": n, "factor_ms": round(ms, 3), "TFLOPs": round(fl / ms / 1e9, 2),
                          "steps": (n + 63) // 64, "us_per_step": round(1e3 * ms / ((n + 63) // 64), 1),
                          "us_per_launch": per, "launches": {k: v["launches"] for k, v in st.items() if v["launches"]}}),
              flush=True)
