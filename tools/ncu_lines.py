"""Per-source-line warp-stall samples from
`ncu -i rep --page source --csv --print-source cuda,sass` output (SASS rows
are attributed to the CUDA line above them)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
acc = collections.Counter()
text = {}
fname, hdr, line = None, None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        line = (fname, r[0])
        text[line] = r[1].strip()
    si = 4
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    if line:
        acc[line] += v
tot = sum(acc.values()) or 1.0
print("total samples", tot)
for (f, ln), v in acc.most_common(n):
    print(f"{v / tot * 100:5.1f}% {f}:{ln} {text.get((f, ln), '')[:100]}")
