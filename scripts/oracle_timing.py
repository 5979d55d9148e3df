"""The CPU baseline at full size (SURVEY §8(d) "oracle timing"): the level-parallel oracle build
(bit-identical to the serial one) on every host core, full C3 and the largest C4 leading samples
(whole ND subtrees); C4 in full is projected from them.  Writes profiles/r02_oracle_timing.json."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402

cores = len(os.sched_getaffinity(0))
out = {"cores": cores, "runs": []}
jobs = [("C3", None), ("C4", 125000), ("C4", 250000), ("C4", 500000)]
for name, ns in jobs:
    p = gen.make(name)
    sub = p if ns is None else gen.leading_submatrix(p, ns)
    o = oracle.Oracle.from_problem(sub)
    t0 = time.perf_counter()
    assert o.factor(threads=cores) == -1
    t = time.perf_counter() - t0
    rec = {"config": name, "cols": sub.n, "flops": o.flops, "seconds": t, "gflops": o.flops / t / 1e9}
    out["runs"].append(rec)
    print(json.dumps(rec), flush=True)
full = gen.make("C4")
c4 = [r for r in out["runs"] if r["config"] == "C4"]
# projection: the largest sample's rate (the rate falls as the sample grows: longer chains)
out["C4_projection_seconds"] = 6.682103420824e12 / (c4[-1]["gflops"] * 1e9)
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("profiles/r02_oracle_timing.json", "w"), indent=1)
print(json.dumps({"C4_projection_seconds": out["C4_projection_seconds"], "cores": cores}))
