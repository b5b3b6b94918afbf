"""Hottest SASS instructions (warp-stall samples) of one kernel of a .ncu-rep.

    python tools/ncu_sass_hot.py report.ncu-rep <kernel-regex> [n]
"""
import csv
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{pat}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
idx = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows if len(r) >= len(hdr) - 1 and r[0].startswith("0x")]
tot = sum(float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
body.sort(key=lambda r: -float(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
print(f"total samples {tot:.0f}")
for r in body[:n]:
    s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100 * s / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:70]:70s} exec={r[idx['Instructions Executed']]}")
