"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 1
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    m = re.search(r"(k_\w+)(<[^>(]*>)?", d["Kernel Name"])
    short = (m.group(1) + (m.group(2) or "")) if m else d["Kernel Name"][:48]
    agg[short][0] += 1
    agg[short][1] += float(d["Metric Value"].replace(",", ""))
total = sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'avg us':>9s} {'ms/frame':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} {v[0]:8d} {v[1] / v[0] / 1e3:9.1f} {v[1] / 1e6 / frames:9.3f} {100 * v[1] / total:5.1f}%")
print(f"{'total':40s} {'':8s} {'':9s} {total / 1e6 / frames:9.3f}")
