"""Summarize an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0, []])
for d in data:
    nm = d['Kernel Name'].split('(')[0][:40]; v = float(d['Metric Value'].replace(',', ''))
    u = d['Metric Unit']
    v = v * 1e3 if u == 'usecond' else v * 1e6 if u == 'msecond' else v
    a = agg[nm]; a[0] += 1; a[1] += v; a[2].append((v / 1e3, d['Grid Size']))
tot = sum(v[1] for v in agg.values())
print("total %.2f ms over %d launches" % (tot / 1e6, len(data)))
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    ts = sorted(x[0] for x in v[2])
    print("%-40s %5d %9.2f ms %5.1f%%  avg %8.1f us  min %.1f  med %.1f  max %.1f" % (k, v[0], v[1] / 1e6, 100 * v[1] / tot, v[1] / v[0] / 1e3, ts[0], ts[len(ts)//2], ts[-1]))
if len(sys.argv) > 2:
    for k, v in agg.items():
        if sys.argv[2] in k:
            print(k, [("%.1f" % t, g) for t, g in v[2][-12:]])
