"""profiles/roofline_traffic.json from an ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum capture of
every SYRK+scatter launch of one C4 factor (scripts/ncu_scatter_only.sh), stamped with the sha256 of the
kernel source it was measured on: bench.py reports roofline.traffic only while that source is unchanged."""
import collections
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "r02_scatter_dram_C4.csv")
rows = list(csv.reader(open(src)))
hdr = next(r for r in rows if "Metric Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
per = collections.defaultdict(dict)
for d in data:
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    if d["Metric Name"] == "gpu__time_duration.sum":
        v = v / 1e3 if u == "usecond" else v if u == "msecond" else v / 1e6
    elif u == "Kbyte":
        v *= 1e3
    elif u == "Mbyte":
        v *= 1e6
    elif u == "Gbyte":
        v *= 1e9
    per[d["ID"]][d["Metric Name"]] = v
n = len(per)
traffic = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in per.values()) / n
ms = sum(x["gpu__time_duration.sum"] for x in per.values())
import gen  # noqa: E402
import paper_2409_14009_b200 as sp  # noqa: E402
with sp.Solver.from_problem(gen.make("C4"), device=-1) as h:
    sym = h.spchol_export_symbolic()
k = sym["sfirst"][1:] - sym["sfirst"][:-1]
m = sym["rows_ptr"][1:] - sym["rows_ptr"][:-1]
t = (m - k).astype(float)
alg = float((8 * t * k + 16 * t * (t + 1) / 2).sum()) / n
kern = open(os.path.join(ROOT, "paper_2409_14009_b200", "csrc", "kernels.cu"), "rb").read()
out = {"config": "C4", "kernel": "syrk_scatter", "launches": n, "traffic_bytes_per_launch": traffic,
       "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": traffic / alg, "ncu_total_ms": ms,
       "kernels_cu_sha256": hashlib.sha256(kern).hexdigest(),
       "source": "profiles/" + os.path.basename(src) + ": ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                 "gpu__time_duration.sum,sm__pipe_fp64_cycles_active... on every SYRK+scatter launch (gemm_kernel<2>) "
                 "of one C4 factor (scripts/stamp_r02b.sh)"}
json.dump(out, open(os.path.join(ROOT, "profiles", "roofline_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
