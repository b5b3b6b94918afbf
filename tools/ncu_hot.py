"""Top instructions by warp-stall samples from `ncu --page source --csv --print-source sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Address":
        cur = (r, [])
        blocks.append(cur)
    elif cur and len(r) == len(cur[0]):
        cur[1].append(r)
for hdr, data in blocks:
    si, src, ad = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Address")
    tot = sum(float(r[si] or 0) for r in data) or 1.0
    print("total samples", tot, "instructions", len(data))
    for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
        print(f"{float(r[si]) / tot * 100:5.1f}% {r[ad]} {r[src][:100]}")
