"""Per-source-line executed warp instructions from
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
        ie = hdr.index("Instructions Executed")
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        line = (fname, r[0])
        text[line] = r[1].strip()
        continue
    try:
        v = float(r[ie] or 0)
    except ValueError:
        continue
    if line:
        acc[line] += v
tot = sum(acc.values())
print(f"total executed {tot:.0f}")
for (f, l), v in acc.most_common(n):
    print(f"{100 * v / tot:5.1f}% {f}:{l} {text.get((f, l), '')[:100]}")
