"""Time spchol_solve_device alone (device-resident b, x; CUDA events) and check the backward error.
Usage: python scripts/solve_bench.py --config C4 [--reps 10]   (SPCHOL_SOLVE_LEGACY=1: old solve)"""
import argparse, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import paper_2409_14009_b200 as sp

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--nrhs", type=int, default=1)
a = ap.parse_args()
p = gen.make(a.config)
h = sp.Solver.from_problem(p, device=0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
h.spchol_set_stream(stream.cuda_stream)
h.spchol_factor()
xs, b = gen.rhs(p)
B = np.repeat(b[:, None], a.nrhs, axis=1).T.copy() if a.nrhs > 1 else b
d_b = torch.from_numpy(np.ascontiguousarray(B)).cuda()
d_x = torch.empty_like(d_b)
h.spchol_solve_device(d_b.data_ptr(), d_x.data_ptr(), a.nrhs)
torch.cuda.synchronize()
x = d_x.cpu().numpy().reshape(a.nrhs, -1)[0]
berr = gen.backward_error(p, x, b)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    h.spchol_solve_device(d_b.data_ptr(), d_x.data_ptr(), a.nrhs)
torch.cuda.synchronize()
e0.record()
for _ in range(a.reps):
    h.spchol_solve_device(d_b.data_ptr(), d_x.data_ptr(), a.nrhs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
nnzL = h.query("NNZ_L")
print(json.dumps({"config": a.config, "legacy": os.environ.get("SPCHOL_SOLVE_LEGACY", "0"), "nrhs": a.nrhs,
                  "solve_ms": round(ms, 3), "GBps_L_twice": round(2 * 8 * nnzL * a.nrhs / (ms / 1e3) / 1e9, 1),
                  "berr": berr, "nnzL": nnzL}))
