"""Summarise an ncu launch list of one solve (scripts/solve_ncu.sh): per-kernel totals and the
sequence of the first solve (between the first two permute launches)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
seq = [(d["Kernel Name"].split("(")[0], float(d["Metric Value"]) / 1e3, d.get("Grid Size", "")) for d in data]
idx = [i for i, s in enumerate(seq) if "permute" in s[0]]
a, b = idx[0], idx[1]
agg = collections.defaultdict(lambda: [0, 0.0])
for s in seq[a:b + 1]:
    agg[s[0]][0] += 1
    agg[s[0]][1] += s[1]
tot = sum(v[1] for v in agg.values())
print(f"one solve: {b - a + 1} launches, {tot:.1f} us (serialized)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:28s} {c:4d} {t:9.1f} us  {100 * t / tot:5.1f}%")
if len(sys.argv) > 2:
    for s in seq[a:b + 1]:
        print(f"  {s[0]:28s} {s[1]:9.1f} us grid {s[2]}")
