"""Time one config's factor (graph) and per-kernel classes for the library in $SPCHOL_LIB."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_2409_14009_b200 as sp

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--block", type=int, default=0)
ap.add_argument("--nograph", action="store_true")
ap.add_argument("--vr", type=int, default=0)
ap.add_argument("--det", type=int, default=0)
a = ap.parse_args()
p = gen.make(a.config)
h = sp.Solver.from_problem(p, block=a.block, use_graph=0 if a.nograph else 1, subtree_streams=a.vr, deterministic=a.det)
F = h.query("FLOPS_EXACT")
for _ in range(2):
    h.spchol_factor()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.Stream()
h.spchol_set_stream(s.cuda_stream)
e0.record(s)
for _ in range(a.steps):
    h.spchol_factor_async()
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
h.spchol_factor_status()
h.spchol_enable_kernel_timing(True)
h.spchol_factor_async()
tr = h.spchol_kernel_trace()
import numpy as np
names = {v: k for k, v in sp.KERNEL_KINDS.items()}
lv = {}
for k, l, n, t in zip(tr["kinds"], tr["levels"], tr["ntasks"], tr["ms"]):
    d = lv.setdefault(int(l), {})
    d[names[int(k)]] = round(d.get(names[int(k)], 0) + float(t), 2)
print(json.dumps({"per_level_ms": lv}))
h.spchol_enable_kernel_timing(True)
for _ in range(a.steps):
    h.spchol_factor_async()
st = {k: h.spchol_kernel_stats(k) for k in sp.KERNEL_KINDS}
out = {"lib": os.environ.get("SPCHOL_LIB", "default"), "nograph": a.nograph, "nola": os.environ.get("SPCHOL_NO_LOOKAHEAD"), "vr": a.vr, "config": a.config, "ms": ms, "tflops": F / ms / 1e9,
       "kernels": {k: {"ms": round(v["ms"] / a.steps, 2), "tf": round(v["flops"] / v["ms"] / 1e9, 2) if v["ms"] else 0}
                   for k, v in st.items() if v["launches"]}}
print(json.dumps(out), flush=True)
