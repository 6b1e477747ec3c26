"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per-kernel totals."""
import csv, collections, sys
path = sys.argv[1]
skip_frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
data = data[int(len(data) * skip_frac):]
agg = collections.OrderedDict(); tot = 0.0
for d in data:
    nm = d['Kernel Name'].split('(')[0].replace('void ', '')[:40]
    v = float(d['Metric Value']) / 1e3
    agg.setdefault(nm, [0.0, 0]); agg[nm][0] += v; agg[nm][1] += 1; tot += v
print(f"{'kernel':40s} {'n':>5s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
for k, (v, c) in sorted(agg.items(), key=lambda t: -t[1][0]):
    print(f"{k:40s} {c:5d} {v:10.1f} {v/c:9.2f} {v/tot:6.3f}")
print(f"{'TOTAL':40s} {len(data):5d} {tot:10.1f}")
